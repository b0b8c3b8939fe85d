# ingest kernel profile: launch list of one C3 load + ncu --set full of the k_bkt kernels
mkdir -p gpurun_out/c3
timeout 300 python tools/profile_load.py --reps 1 > gpurun_out/c3/pl.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3/launches.csv python tools/profile_load.py --reps 1 > gpurun_out/c3/ncu1.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bkt -c 8 -o gpurun_out/c3/bkt python tools/profile_load.py --reps 1 > gpurun_out/c3/ncu2.log 2>&1; echo "full rc=$?"
