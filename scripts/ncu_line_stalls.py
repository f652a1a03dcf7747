"""Warp-stall samples of one ncu-captured kernel aggregated per CUDA source line.

    python scripts/ncu_line_stalls.py <rep.ncu-rep> <kernel-regex> <launch-index> <lib.so> [top]

The SASS view of the ncu source page carries the samples per instruction address; the line
of each instruction comes from `nvdisasm -g` of the same kernel in the shipped library
(instruction offset = address - the kernel's first address).  Prints the top lines with
their dominant stall reasons.
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def line_map(lib, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        funcs = {}
        cur_fn, cur_line, cur_file = None, None, None
        for ln in out.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"^(\S+):\s*$", ln)
            if ln.startswith(".text.") or re.match(r"\s*\.section\s+\.text\.", ln):
                pass
            m = re.search(r"\.text\.([^\s,\"]+)", ln)
            if m and ("section" in ln):
                cur_fn = m.group(1)
                funcs.setdefault(cur_fn, {})
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur_file, cur_line = os.path.basename(m.group(1)), int(m.group(2))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
            if m and cur_fn is not None:
                funcs[cur_fn][int(m.group(1), 16)] = (cur_file, cur_line)
        for fn, mp in funcs.items():
            if re.search(mangled_hint, fn) and mp:
                return fn, mp
    return None, {}


def main():
    rep, kern, skip, lib = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr, data = rows[hi], [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
    col = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    base = int(data[0][0], 16)
    fn, mp = line_map(lib, kern)
    print("function:", fn, "instructions mapped:", len(mp))
    f = lambda r, h: float(r[col[h]] or 0)  # noqa: E731
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    per_line = defaultdict(lambda: defaultdict(float))
    for r in data:
        off = int(r[0], 16) - base
        key = mp.get(off, ("?", -1))
        d = per_line[key]
        d["all"] += f(r, "Warp Stall Sampling (All Samples)")
        for s in stalls:
            d[s] += f(r, s)
    items = sorted(per_line.items(), key=lambda kv: -kv[1]["all"])[:top]
    for (fl, ln), d in items:
        reasons = sorted(((k, v) for k, v in d.items() if k != "all" and v > 0), key=lambda kv: -kv[1])[:3]
        rs = ", ".join(f"{k[6:]}={100 * v / d['all']:.0f}%" for k, v in reasons)
        print(f"{100 * d['all'] / tot:5.1f}%  {fl}:{ln:<5d} {rs}")


if __name__ == "__main__":
    main()
