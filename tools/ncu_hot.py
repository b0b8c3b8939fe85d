"""Summarise an ncu report's hot source lines (stall samples), CUDA-source correlated."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
S, I = 4, 7  # columns: Line No, Source, Address, Source, stall(all), stall(not issued), #samples, instr executed
def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0
data = [r for r in rows[hdr_i + 1:] if len(r) > 8 and r[0].isdigit()]
tot = sum(iv(r[S]) for r in data) or 1
totI = sum(iv(r[I]) for r in data) or 1
print("samples", tot, "warp-instr", totI)
for r in sorted(data, key=lambda r: -iv(r[S]))[:n]:
    print(f"{iv(r[S])/tot*100:5.1f}% I={iv(r[I])/totI*100:5.1f}% L{r[0]:>4} {r[1].strip()[:95]}")
