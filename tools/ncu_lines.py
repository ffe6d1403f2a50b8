"""Per-source-line warp-stall samples of one kernel from an ncu report.

ncu's SASS source page (--page source --print-source sass --csv) carries the
PC-sampling counts per instruction; nvdisasm -g on the same cubin maps each
instruction offset to a CUDA source line (the library is built with
-lineinfo).  Usage:

    ncu -i rep.ncu-rep --page source --csv --print-source sass > k.csv
    python tools/ncu_lines.py k.csv paper_2106_11594_b200/librgb.so <kernel-substring> [top]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(path, column="Warp Stall Sampling (All Samples)"):
    rows = list(csv.reader(open(path)))
    kname = rows[0][1] if len(rows[0]) > 1 else ""
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    iall = h.index(column)
    data = [(int(r[ia], 16), r[isrc].strip(), float(r[iall] or 0)) for r in rows[2:] if r[ia].startswith("0x")]
    base = data[0][0]
    return kname, [(a - base, s, n) for a, s, n in data]


def line_map(so, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True, check=True)
    out = {}
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin") or "-" in f:
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        func, line, fmap = None, None, {}
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                func, line, fmap = m.group(1), None, {}
                out[func] = fmap
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                line = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and func is not None:
                fmap[int(m.group(1), 16)] = line
    cands = [k for k in out if kernel_sub in k]
    return cands, out


def main():
    csvp, so, sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    # RGB_NCU_COLUMN="Instructions Executed" ranks lines by executed instructions instead
    kname, samples = sass_samples(csvp, os.environ.get("RGB_NCU_COLUMN", "Warp Stall Sampling (All Samples)"))
    cands, maps = line_map(so, sub)
    # pick the candidate whose instruction count matches the sampled kernel
    best = max(cands, key=lambda k: -abs(len(maps[k]) - len(samples)))
    fmap = maps[best]
    agg, tot = {}, 0.0
    for off, s, n in samples:
        key = fmap.get(off, ("?", 0))
        agg[key] = agg.get(key, 0.0) + n
        tot += n
    print(f"{kname}\nmapped with {best} ({len(fmap)} instr vs {len(samples)} sampled); samples {tot:.0f}")
    src_cache = {}
    for (f, l), n in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        text = ""
        for root in ("paper_2106_11594_b200/csrc", "."):
            p = os.path.join(root, f)
            if os.path.exists(p):
                src_cache.setdefault(p, open(p).read().splitlines())
                text = src_cache[p][l - 1].strip() if 0 < l <= len(src_cache[p]) else ""
                break
        print(f"{100 * n / tot:5.1f}%  {f}:{l}  {text[:90]}")


if __name__ == "__main__":
    main()
