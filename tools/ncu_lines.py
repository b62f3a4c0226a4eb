"""Aggregate an ncu --page source --csv --print-source cuda,sass export by
(file, line): instructions executed, thread instructions, warp-stall samples.
python tools/ncu_lines.py export.csv [top] [kernel-substring]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ksub = sys.argv[3] if len(sys.argv) > 3 else ""
agg, thr, smp, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
cur_file, cur_fn = "?", ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No" or ksub not in cur_fn:
        continue
    if r[0] and len(r) > 8:   # a CUDA source line (its SASS rows follow with an empty line number)
        try:
            ie, ti, s = float(r[7] or 0), float(r[8] or 0), float(r[4] or 0)
        except ValueError:
            continue
        k = (cur_file, int(r[0]))
        src[k] = r[1].strip()[:90]
        agg[k] += ie
        thr[k] += ti
        smp[k] += s
T, TT, TS = sum(agg.values()) or 1, sum(thr.values()) or 1, sum(smp.values()) or 1
print(f"warp-instructions {T:.4g}  thread-instructions {TT:.4g}  samples {TS:.0f}")
print("by file:", {f: round(sum(v for k, v in agg.items() if k[0] == f) / T * 100, 1) for f in {k[0] for k in agg}})
for k, v in sorted(agg.items(), key=lambda kv: -(smp[kv[0]] + kv[1] / T * TS))[:top]:
    print(f"{v / T * 100:5.1f}%i {thr[k] / TT * 100:5.1f}%t {smp[k] / TS * 100:5.1f}%s {k[0]}:{k[1]} {src[k]}")
