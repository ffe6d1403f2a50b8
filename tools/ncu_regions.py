"""Warp-stall samples of one kernel per source line of a chosen file, with the
stall reasons, attributing inlined helpers (mma, shuffles, rcp64) to the line of
the CALLER in that file (nvdisasm -gi line tables).

    ncu -i rep.ncu-rep --page source --csv --print-source sass > k.csv
    python tools/ncu_regions.py k.csv paper_2106_11594_b200/librgb.so <kernel-substring> rgb_panel.cu [ranges]
ranges: name:first-last,... (source lines of the file) to aggregate regions.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ia = h.index("Address")
    reasons = [c for c in h if c.startswith("stall_") and "(Not Issued)" not in c]
    idx = {c: h.index(c) for c in reasons}
    iall = h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if not r[ia].startswith("0x"):
            continue
        data.append((int(r[ia], 16), float(r[iall] or 0), {c: float(r[i] or 0) for c, i in idx.items()}))
    base = data[0][0]
    return [(a - base, n, d) for a, n, d in data], reasons


def line_map(so, kernel_sub, fname, ninstr):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True, check=True)
    best = None
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin") or "-" in f:
            continue
        txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        func, cur, fmap = None, None, None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                if func and kernel_sub in func and (best is None or abs(len(fmap) - ninstr) < abs(len(best) - ninstr)):
                    best = fmap
                func, cur, fmap = m.group(1), None, {}
                continue
            if "//##" in ln and fname in ln:
                # outermost occurrence of the file in this line-info record (caller side)
                ms = re.findall(r'File "[^"]*' + re.escape(fname) + r'", line (\d+)', ln)
                if ms:
                    # outermost by default; RGB_NCU_INNER=1: the innermost line of this file
                    cur = int(ms[0] if os.environ.get("RGB_NCU_INNER") else ms[-1])
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and func is not None:
                fmap[int(m.group(1), 16)] = cur
        if func and kernel_sub in func and (best is None or abs(len(fmap) - ninstr) < abs(len(best) - ninstr)):
            best = fmap
    return best


def main():
    csvp, so, sub, fname = sys.argv[1:5]
    ranges = []
    if len(sys.argv) > 5:
        for part in sys.argv[5].split(","):
            nm, rg = part.split(":")
            a, b = rg.split("-")
            ranges.append((nm, int(a), int(b)))
    samples, reasons = load(csvp)
    fmap = line_map(so, sub, fname, len(samples))
    tot = sum(n for _, n, _ in samples)
    agg = {}
    for off, n, d in samples:
        ln = fmap.get(off)
        nm = "other"
        for rn, a, b in ranges:
            if ln is not None and a <= ln <= b:
                nm = rn
                break
        e = agg.setdefault(nm, [0.0, {}])
        e[0] += n
        for c, v in d.items():
            e[1][c] = e[1].get(c, 0.0) + v
    for nm, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        top = sorted(d.items(), key=lambda kv: -kv[1])[:5]
        print(f"{nm:12s} {100 * n / tot:5.1f}%  " + "  ".join(f"{c[6:]} {100 * v / max(n, 1):.0f}%" for c, v in top))


if __name__ == "__main__":
    main()


def lines(csvp, so, sub, fname, a, b, top=25):
    """Top source lines of [a, b] by samples, with executed warp instructions."""
    rows = list(csv.reader(open(csvp)))
    h = rows[1]
    ia, iall, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [(int(r[ia], 16), float(r[iall] or 0), float(r[iex] or 0)) for r in rows[2:] if r[ia].startswith("0x")]
    base = data[0][0]
    fmap = line_map(so, sub, fname, len(data))
    agg = {}
    for addr, n, ex in data:
        ln = fmap.get(addr - base)
        if ln is None or not a <= ln <= b:
            continue
        e = agg.setdefault(ln, [0.0, 0.0, 0])
        e[0] += n
        e[1] += ex
        e[2] += 1
    src = open(os.path.join("paper_2106_11594_b200/csrc", fname)).read().splitlines()
    tot = sum(v[0] for v in agg.values())
    for ln, (n, ex, ni) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * n / tot:5.1f}%  L{ln:4d} sass {ni:3d} exec {ex:12.0f}  {src[ln - 1].strip()[:80]}")
