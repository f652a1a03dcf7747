"""Instruction mix of a kernel's SASS per source-line range (nvdisasm -g output).

    python scripts/sass_lines.py <kernel.sass> <file-substring> <line-lo> <line-hi>
"""
import re
import sys
from collections import Counter


def main():
    path, fsub, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    cur = None
    mix = Counter()
    n = 0
    for ln in open(path):
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = int(m.group(2)) if fsub in m.group(1) else None
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(.*?);", ln)
        if m and cur is not None and lo <= cur <= hi:
            toks = m.group(1).split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            mix[op] += 1
            n += 1
    print(n, "instructions")
    for op, c in mix.most_common(30):
        print(f"{c:6d} {op}")


if __name__ == "__main__":
    main()
