"""Build librgb.so in-tree with nvcc for sm_100a (no torch in the ABI)."""

from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librgb.so")
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = [*ARCH_FLAGS, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
NVCC_FLAGS = [*COMPILE_FLAGS, "-shared"]  # one-command form (documentation / debugging)


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
        os.path.join(ROOT, "include", "rgb.h")]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force=False, log=None):
    """Compile every csrc/*.cu to an object in parallel (-rdc off, whole-program
    per file), then link librgb.so."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        jobs.append((src, obj, [nvcc, *COMPILE_FLAGS, "-c", "-o", obj, src]))

    def run(job):
        return job, subprocess.run(job[2], capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
        results = list(pool.map(run, jobs))
    link = [nvcc, *ARCH_FLAGS, "-shared", "-o", LIB, *[j[1] for j in jobs]]
    lres = subprocess.run(link, capture_output=True, text=True) if all(r.returncode == 0 for _, r in results) else None
    if log is not None:
        with open(log, "w") as f:
            for job, res in results:
                f.write(" ".join(job[2]) + "\n" + res.stdout + res.stderr)
            if lres is not None:
                f.write(" ".join(link) + "\n" + lres.stdout + lres.stderr)
    for job, res in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(job[0])}:\n" + res.stderr[-4000:])
    if lres.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + lres.stderr[-4000:])
    return LIB


if __name__ == "__main__":
    build(force=True, log=os.path.join(HERE, "build.log"))
    print(LIB)


PEAK_SRC = os.path.join(ROOT, "tools", "fp64_peak.cu")
PEAK_LIB = os.path.join(ROOT, "tools", "libfp64peak.so")


def build_peak_probe(force=False):
    """tools/libfp64peak.so: the live fp64 peak probe bench.py uses as the
    roofline denominator (MEASURED_PEAKS.json has no fp64 entry)."""
    if not force and os.path.exists(PEAK_LIB) and os.path.getmtime(PEAK_LIB) > os.path.getmtime(PEAK_SRC):
        return PEAK_LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
           "-o", PEAK_LIB, PEAK_SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-4000:])
    return PEAK_LIB


DEMO_SRC = os.path.join(ROOT, "examples", "rgb_demo.c")
DEMO_BIN = os.path.join(ROOT, "examples", "rgb_demo")


def build_demo(force=False):
    """The plain-C consumer of the ABI (examples/rgb_demo.c), linked against librgb.so."""
    if not force and os.path.exists(DEMO_BIN) and os.path.getmtime(DEMO_BIN) > os.path.getmtime(DEMO_SRC):
        return DEMO_BIN
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-O2", "-o", DEMO_BIN, DEMO_SRC, "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(cuda, "include"), "-L" + HERE, "-lrgb", "-L" + os.path.join(cuda, "lib64"),
           "-lcudart", "-lm", "-Wl,-rpath,$ORIGIN/../paper_2106_11594_b200"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("demo build failed:\n" + res.stderr[-2000:])
    return DEMO_BIN
