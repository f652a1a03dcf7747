"""Aggregate ncu per-instruction warp-stall samples (source page, SASS view).

    python scripts/ncu_sass_stalls.py gpurun_out/x.ncu-rep <kernel-regex> [launch-index] [top]

Prints stall totals per reason, per opcode, and the top instructions with their dominant
stall reasons (needs a capture with --set full --import-source on).
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kern, "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr, data = rows[hi], [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
    col = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    f = lambda r, h: float(r[col[h]] or 0)  # noqa: E731
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"{len(data)} instructions, {tot:.0f} samples")
    by_reason = {s: sum(f(r, s) for r in data) for s in stalls}
    print("by reason:", ", ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in
                                 sorted(by_reason.items(), key=lambda kv: -kv[1]) if v > 0))
    by_op = defaultdict(float)
    for r in data:
        by_op[r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]] += f(
            r, "Warp Stall Sampling (All Samples)")
    print("by opcode:", ", ".join(f"{k}={100 * v / tot:.1f}%" for k, v in
                                 sorted(by_op.items(), key=lambda kv: -kv[1])[:15]))
    idx = sorted(range(len(data)), key=lambda i: -f(data[i], "Warp Stall Sampling (All Samples)"))[:top]
    for i in sorted(idx):
        r = data[i]
        s = sorted(((f(r, h), h[6:]) for h in stalls), reverse=True)[:3]
        print(f"{i:5d} {100 * f(r, 'Warp Stall Sampling (All Samples)') / tot:5.1f}%  "
              f"{r[1].strip()[:60]:60s} " + " ".join(f"{n}={v:.0f}" for v, n in s if v > 0))


if __name__ == "__main__":
    main()
