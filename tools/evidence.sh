#!/bin/bash
# Round-end evidence (run under gpurun): bench lines (C3 triangles, C4 4-cliques),
# the oracle reference arm, per-config table, launch list of the bench command,
# ncu --set full of the count kernels, the oracle by the paper's protocol.
# Outputs in gpurun_out/ev/.
mkdir -p gpurun_out/ev
E=gpurun_out/ev
nproc > $E/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $E/nproc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $E/bench.json 2> $E/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --query k4 --steps 10 --warmup 3 > $E/bench_k4.json 2> $E/bench_k4.err; echo "bench k4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $E/bench_ref.json 2> $E/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/bench_configs.py --k4 > $E/configs.jsonl 2> $E/configs.err; echo "configs rc=$?"
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $E/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $E/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $E/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/profile_count.py --reps 1 > $E/pc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tri -c 3 -o $E/tri_C3 \
  python tools/profile_count.py --reps 1 > $E/ncu_tri.log 2>&1; echo "ncu tri rc=$?"
timeout 300 python tools/profile_count.py --config C4 --query k4 --reps 1 > $E/pc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_k4 -c 6 -o $E/k4_C4 \
  python tools/profile_count.py --config C4 --query k4 --reps 1 > $E/ncu_k4.log 2>&1; echo "ncu k4 rc=$?"
timeout 1800 python tools/oracle_protocol.py C1 C2 C3 C4 > $E/oracle_protocol.jsonl 2> $E/oracle_protocol.err; echo "oracle rc=$?"
