"""profiles/traffic.json from `ncu --set full` reports of the count kernels:
dram__bytes_read.sum + dram__bytes_write.sum summed over the launches of one
count call.  Usage: traffic_from_ncu.py [--keep OLD.json] NAME=REPORT ... > profiles/traffic.json
(NAME e.g. tri_C3, k4_C4, tri_C5; entries of OLD.json that are not re-measured are kept)."""
import csv
import json
import math
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    tot, kernels, missing = 0.0, [], []
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
        kernels.append(name)
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                v = float("nan")
            if math.isnan(v):
                if name not in missing:
                    missing.append(name)  # ncu returned no value for this launch
                continue
            tot += v * SCALE[units[i]]
    return int(round(tot)), kernels, missing


args = sys.argv[1:]
out = {}
if args and args[0] == "--keep":
    out = json.load(open(args[1]))
    args = args[2:]
out["source"] = ("ncu --set full --clock-control none (cold caches) via tools/evidence.sh; dram__bytes_read.sum + "
                 "dram__bytes_write.sum summed over the launches of one count call; reports summarised in "
                 "profiles/r2_count_kernels_v4.md (entries not listed there: earlier captures, see profiles/README.md)")
for a in args:
    name, rep = a.split("=", 1)
    b, k, miss = dram_bytes(rep)
    out[name + "_bytes_per_launch"] = b
    out[name.split("_")[0] + "_kernels" if name in ("tri_C3", "k4_C4") else name + "_kernels"] = k
    if miss:
        out[name + "_kernels_without_dram_counters"] = miss
print(json.dumps(out, indent=1))
