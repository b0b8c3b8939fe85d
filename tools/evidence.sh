#!/bin/bash
# Round-end evidence (run under gpurun): bench lines (C3 triangles, C4 4-cliques),
# the oracle reference arm, per-config table, launch list of the bench command,
# ncu --set full of the count kernels (C3 / C5 triangles, C4 4-cliques) and of the ingest
# kernels (C3), the intersection microbenchmarks, the oracle by the paper's protocol.
# Outputs in gpurun_out/ev/ (the .ncu-rep files stay in /tmp on the box except tri_C3:
# gpurun merges at most 64 MiB back; their summaries are written here).
mkdir -p gpurun_out/ev /tmp/ev_reps
E=gpurun_out/ev; R=/tmp/ev_reps
nproc > $E/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $E/nproc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $E/bench.json 2> $E/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --query k4 --steps 10 --warmup 3 > $E/bench_k4.json 2> $E/bench_k4.err; echo "bench k4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $E/bench_ref.json 2> $E/bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/bench_configs.py --k4 > $E/configs.jsonl 2> $E/configs.err; echo "configs rc=$?"
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $E/bench_small.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $E/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $E/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/profile_count.py --reps 1 > $E/pc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tri -c 3 -o $R/tri_C3 \
  python tools/profile_count.py --reps 1 > $E/ncu_tri.log 2>&1; echo "ncu tri rc=$?"
timeout 300 python tools/profile_count.py --config C4 --query k4 --reps 1 > $E/pc.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_k4 -c 6 -o $R/k4_C4 \
  python tools/profile_count.py --config C4 --query k4 --reps 1 > $E/ncu_k4.log 2>&1; echo "ncu k4 rc=$?"
timeout 900 python tools/profile_count.py --config C5 --reps 1 > $E/pc5.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_tri -c 5 -o $R/tri_C5 \
  python tools/profile_count.py --config C5 --reps 1 > $E/ncu_tri5.log 2>&1; echo "ncu c5 rc=$?"
# --set full returns no counter values for the C5 mid-class CTA kernel (time only): capture it
# again with an explicit metric list + the SourceCounters section, on one stream
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__inst_executed.sum,lts__t_bytes.sum
EH_TEST_TRI_SERIAL=1 timeout 1500 ncu --metrics $M --section SourceCounters --clock-control none --import-source on \
  --kernel-id ::regex:k_tri_cta:2 -o $R/tri_C5_mid -f python tools/profile_count.py --config C5 --reps 1 > $E/ncu_tri5_mid.log 2>&1; echo "ncu c5 mid rc=$?"
timeout 300 python tools/profile_load.py --reps 2 > $E/pl.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_bkt|k_scatter|k_seg|k_fill|k_layout|k_rank|k_max_id|k_radix|k_deg" -c 60 -o $R/load_C3 \
  python tools/profile_load.py --reps 1 > $E/ncu_load.log 2>&1; echo "ncu load rc=$?"
for r in tri_C3 k4_C4 tri_C5 tri_C5_mid load_C3; do python tools/ncu_summary.py $R/$r.ncu-rep $r > $E/$r.summary.md 2>> $E/summary.err; done
for spec in "tri_C3 k_tri_cta" "tri_C3 k_tri_warp" "tri_C5 k_tri_cta" "tri_C5_mid k_tri_cta" "tri_C5 k_tri_warp" "k4_C4 k_k4_cta" "k4_C4 k_k4_warp" \
  "load_C3 k_bkt_part" "load_C3 k_bkt_dedup" "load_C3 k_scatter_col"; do set -- $spec
  { echo "#### $1 $2"; echo '```'; python tools/ncu_hot.py $R/$1.ncu-rep 16 "$2"; echo '```'; echo; } >> $E/hot_lines.md 2>> $E/summary.err; done
python tools/traffic_from_ncu.py --keep profiles/traffic.json tri_C3=$R/tri_C3.ncu-rep k4_C4=$R/k4_C4.ncu-rep tri_C5=$R/tri_C5.ncu-rep > $E/traffic.json 2>> $E/summary.err
cp $R/tri_C3.ncu-rep $E/
EH_TIMING=1 timeout 300 python tools/profile_load.py --reps 3 2>&1 | grep timing | tail -1 > $E/load_phases_C3.txt
timeout 900 python tools/intersect_bench.py E2 E16a E16b > $E/intersect_micro.jsonl 2> $E/intersect_micro.err; echo "micro rc=$?"
timeout 1800 python tools/oracle_protocol.py C1 C2 C3 C4 > $E/oracle_protocol.jsonl 2> $E/oracle_protocol.err; echo "oracle rc=$?"
