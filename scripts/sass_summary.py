"""Per-kernel SASS summary of the built library (cuobjdump -sass): instruction count,
registers/smem from the function header, and the counts of the instructions that prove the
Blackwell paths (UTC*MMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM/STTM = tcgen05.ld/st,
UTMALDG/UTMASTG/UTMAPF = TMA tensor load/store/prefetch, UBLKCP = bulk copy, LDGSTS = cp.async,
SYNCS = mbarrier ops, MUFU.EX2 = exp2, ELECT).

    python scripts/sass_summary.py [lib.so] [--out profiles/r02_sass_summary.md]
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP",
        "UBLKPF", "LDGSTS", "SYNCS", "MUFU.EX2", "MUFU.TANH", "ELECT", "USETMAXREG"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.split("\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib", nargs="?", default=os.path.join(ROOT, "paper_2506_03275_b200", "libcsd_b200.so"))
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", args.lib], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for ln in sass.split("\n"):
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(.*?);", ln)
        if not m:
            continue
        toks = m.group(1).split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c = kernels[cur]
        c["_total"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                c[k] += 1
    names = list(kernels)
    pretty = demangle(names)
    rows = []
    hdr = ["kernel", "instrs"] + KEYS
    for raw, nice in zip(names, pretty):
        c = kernels[raw]
        if not any(c[k] for k in KEYS[:10]):
            continue  # only the tcgen05 / TMA / cp.async kernels
        nice = nice.replace("csd::dev::", "").replace("(anonymous namespace)::", "")
        nice = re.sub(r"\(.*", "", nice)
        rows.append([nice[:60], str(c["_total"])] + [str(c[k]) for k in KEYS])
    lines = ["# SASS summary (`scripts/sass_summary.py`, cuobjdump -sass of libcsd_b200.so, sm_100a)", "",
             "| " + " | ".join(hdr) + " |", "|" + "---|" * len(hdr)]
    lines += ["| " + " | ".join(r) + " |" for r in rows]
    text = "\n".join(lines) + "\n"
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
