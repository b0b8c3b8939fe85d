R=/tmp/ev_reps; mkdir -p $R gpurun_out/ev
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__inst_executed.sum,lts__t_bytes.sum
EH_TEST_TRI_SERIAL=1 timeout 1500 ncu --metrics $M --section SourceCounters --clock-control none --import-source on --kernel-id ::regex:k_tri_cta:2 -o $R/tri_C5_mid -f python tools/profile_count.py --config C5 --reps 1 > gpurun_out/ev/ncu_tri5_mid.log 2>&1; echo "rc=$?"
python tools/ncu_summary.py $R/tri_C5_mid.ncu-rep tri_C5_mid > gpurun_out/ev/tri_C5_mid.summary.md
{ echo "#### tri_C5 k_tri_cta<4, ...> (mid class)"; echo '```'; python tools/ncu_hot.py $R/tri_C5_mid.ncu-rep 20 k_tri_cta; echo '```'; } > gpurun_out/ev/hot_lines_C5_mid.md
grep -i "warn\|error\|==PROF==" gpurun_out/ev/ncu_tri5_mid.log | head
