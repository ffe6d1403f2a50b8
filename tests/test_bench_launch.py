"""bench.py's own rank launcher (`python bench.py --gpus N` without torchrun):
N processes with the torchrun environment, a working gloo rendezvous between
them, failure propagation, and the WORLD_SIZE / --gpus consistency check.
The GPU half (two ranks of the real bench sharing one B200) is in
test_gpu_parity.py::test_bench_two_ranks_equal_one_rank."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


WORKER = r"""
import os, sys
import torch, torch.distributed as dist
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
t = torch.tensor([float(r + 1)])
dist.all_reduce(t)
assert int(os.environ["LOCAL_RANK"]) == r and os.environ["MASTER_ADDR"] == "127.0.0.1"
open(os.path.join(sys.argv[1], f"rank{r}"), "w").write(f"{w} {t.item():g}")
dist.destroy_process_group()
"""


def test_launch_ranks_sets_torchrun_env_and_rendezvous(tmp_path):
    rc = bench.launch_ranks(3, [sys.executable, "-c", WORKER, str(tmp_path)])
    assert rc == 0
    got = sorted(p.name for p in tmp_path.iterdir())
    assert got == ["rank0", "rank1", "rank2"]
    for p in tmp_path.iterdir():
        assert p.read_text() == "3 6"  # world size 3, all-reduce of 1 + 2 + 3


def test_launch_ranks_propagates_failure_and_stops_peers():
    # rank 1 fails at once; rank 0 would block in the rendezvous forever
    code = ("import os, sys, time\n"
            "sys.exit(3) if os.environ['RANK'] == '1' else time.sleep(600)")
    rc = bench.launch_ranks(2, [sys.executable, "-c", code])
    assert rc == 3


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE=2" in p.stderr


@pytest.mark.parametrize("gpus", [1, 2])
def test_reference_arm_prints_one_line_on_rank0_only(gpus):
    """--impl reference: rank 0 alone times the CPU reference; other ranks exit 0."""
    env = dict(os.environ, RANK="1", WORLD_SIZE=str(gpus), LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", str(gpus)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == ""
