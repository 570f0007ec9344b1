"""Split an ncu source-page CSV (--page source --csv --print-source sass) into
address ranges and print instructions / stall reasons per range.

    python tools/ncu_regions.py src.csv name:lo:hi [name:lo:hi ...]   (hex offsets)
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[1]
    ai, ei = h.index("Address"), h.index("Instructions Executed")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ri = [h.index(c) for c in reasons]
    seq = []
    for r in rows[2:]:
        try:
            seq.append((int(r[ai], 16), int(r[ei]), [int(r[i]) for i in ri]))
        except (ValueError, IndexError):
            continue
    base = seq[0][0]
    tot = sum(x[1] for x in seq)
    stot = sum(sum(x[2]) for x in seq)
    for spec in sys.argv[2:]:
        name, lo, hi = spec.split(":")
        lo, hi = int(lo, 16), int(hi, 16)
        sel = [x for x in seq if lo <= x[0] - base < hi]
        c = sum(x[1] for x in sel)
        st = [sum(x[2][k] for x in sel) for k in range(len(reasons))]
        s = sum(st)
        top = sorted(zip(st, reasons), reverse=True)[:5]
        print(f"{name:10s} instr {c / tot * 100:5.1f}%  stalls {s / max(stot, 1) * 100:5.1f}%  " +
              " ".join(f"{n[6:]}={v / max(s, 1) * 100:.0f}%" for v, n in top))


if __name__ == "__main__":
    main()
