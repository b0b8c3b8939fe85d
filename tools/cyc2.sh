# GPU iteration: parity tests (optionally -k), bench with phase timing, configs
mkdir -p gpurun_out/c2
K=${1:-}
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/c2/pytest.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c2/pytest.log 2>&1; fi
echo "pytest rc=$?" >> gpurun_out/c2/pytest.log; tail -3 gpurun_out/c2/pytest.log
EH_TIMING=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c2/bench.json 2> gpurun_out/c2/bench.err; echo "bench rc=$?"
EH_TEST_DEDUP=sort EH_TIMING=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c2/bench_sort.json 2> gpurun_out/c2/bench_sort.err; echo "bench sort rc=$?"
timeout 900 python tools/bench_configs.py > gpurun_out/c2/configs.jsonl 2> gpurun_out/c2/configs.err; echo "configs rc=$?"
