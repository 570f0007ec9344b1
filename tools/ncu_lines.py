"""Per-source-line instruction / stall-sample table of one ncu report's
source page (ncu -i X --page source --csv --print-source cuda,sass):
    python tools/ncu_lines.py src.csv [top]
Prints the hottest CUDA lines by warp-instructions executed and by stall
samples, and the SASS opcode mix of the kernel."""
import csv, sys, collections
rows = csv.reader(open(sys.argv[1]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
lines = []
ops = collections.Counter()
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:   # CUDA line aggregate
        try:
            lines.append((fname, int(r[0]), r[1].strip()[:70], int(r[4]), int(r[7])))
        except ValueError:
            pass
    elif r[2] not in ("", "...") and r[7] not in ("-", ""):
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        ops[op.split(".")[0]] += int(r[7])
tot_i = sum(l[4] for l in lines) or 1
tot_s = sum(l[3] for l in lines) or 1
print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
print("--- by instructions")
for l in sorted(lines, key=lambda x: -x[4])[:top]:
    print(f"{l[0]:>16s}:{l[1]:<5d} {l[4] / tot_i * 100:5.1f}% inst {l[3] / tot_s * 100:5.1f}% stall  {l[2]}")
print("--- by stall samples")
for l in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{l[0]:>16s}:{l[1]:<5d} {l[4] / tot_i * 100:5.1f}% inst {l[3] / tot_s * 100:5.1f}% stall  {l[2]}")
print("--- SASS opcode mix")
to = sum(ops.values()) or 1
for o, n in ops.most_common(30):
    print(f"{o:12s} {n / to * 100:5.1f}%")
