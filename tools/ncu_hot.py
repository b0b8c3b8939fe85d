"""Hot CUDA-source lines (stall samples) per kernel of an ncu report.
Usage: ncu_hot.py REPORT [N] [kernel-substring]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilt = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0
sections, cur, fn = [], None, ""
for r in rows:
    if r and r[0] == "Function Name":
        fn = r[1]
    elif r and r[0] == "Line No":
        cur = (fn, []); sections.append(cur)
    elif cur is not None and len(r) > 8 and r[0].isdigit():
        cur[1].append(r)
agg = {}
for fn, data in sections:
    if kfilt and kfilt not in fn:
        continue
    for r in data:
        key = (fn.split("(")[0].split("::")[-1], r[0], r[1].strip()[:90])
        a = agg.setdefault(key, [0, 0])
        a[0] += iv(r[4]); a[1] += iv(r[7])
tot = sum(v[0] for v in agg.values()) or 1
totI = sum(v[1] for v in agg.values()) or 1
print("samples", tot, "warp-instr", totI)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{v[0]/tot*100:5.1f}% I={v[1]/totI*100:5.1f}% {k[0][:12]} L{k[1]:>4} {k[2]}")
