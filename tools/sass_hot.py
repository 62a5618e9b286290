"""Summarize an `ncu --page source --csv --print-source sass` export: instruction mix,
stall samples by opcode, and the hottest code regions.

    python tools/sass_hot.py gpurun_out/x_sass.csv [--window 100]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    win = int(sys.argv[sys.argv.index("--window") + 1]) if "--window" in sys.argv else 100
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    iE, iS = hdr.index("Instructions Executed"), hdr.index("Source")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    seq = []
    for r in rows[2:]:
        try:
            n = int(r[iE])
        except (ValueError, IndexError):
            continue
        src = r[iS].strip()
        tok = src.split()
        op = (tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")).split(".")[0]
        seq.append((n, int(r[iW] or 0), op, src))
    tot = sum(s[0] for s in seq)
    st = sum(s[1] for s in seq)
    byop, stall = collections.Counter(), collections.Counter()
    for n, w, op, _ in seq:
        byop[op] += n
        stall[op] += w
    print(f"warp instructions {tot}, stall samples {st}")
    for k, v in byop.most_common(16):
        print(f"  {k:8s} {v:10d} {100 * v / tot:5.1f}%   stall {100 * stall[k] / max(st, 1):5.1f}%")
    print("regions (index, instr, stall%, first op):")
    for i in range(0, len(seq), win):
        ch = seq[i:i + win]
        ni, wi = sum(c[0] for c in ch), sum(c[1] for c in ch)
        if ni:
            print(f"  {i:5d} {ni:10d} {100 * wi / max(st, 1):5.1f}%  {ch[0][3][:50]}")


if __name__ == "__main__":
    main()
