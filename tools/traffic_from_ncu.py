"""profiles/traffic.json from `ncu --set full` reports of the count kernels:
dram__bytes_read.sum + dram__bytes_write.sum summed over the launches of one
count call.  Usage: traffic_from_ncu.py TRI_REP PV_REP K4_REP > profiles/traffic.json"""
import csv
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def dram_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    tot, kernels = 0.0, []
    for r in data:
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i].replace(",", "")) * SCALE[units[i]]
        kernels.append(r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1])
    return int(round(tot)), kernels


tri, kt = dram_bytes(sys.argv[1])
pv, kp = dram_bytes(sys.argv[2])
k4, kk = dram_bytes(sys.argv[3])
print(json.dumps({
    "source": "ncu --set full --clock-control none (cold caches) via tools/evidence.sh; dram__bytes_read.sum + "
              "dram__bytes_write.sum summed over the launches of one count call; reports summarised in "
              "profiles/r1_count_kernels_v5.md",
    "tri_C3_bytes_per_launch": tri, "tri_kernels": kt,
    "pv_C3_bytes_per_launch": pv, "pv_kernels": kp,
    "k4_C4_bytes_per_launch": k4, "k4_kernels": kk}, indent=1))
