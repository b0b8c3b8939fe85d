mkdir -p gpurun_out/c1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/c1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/c1/bench.json 2> gpurun_out/c1/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --query k4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1/bench_k4.json 2> gpurun_out/c1/bench_k4.err; echo "k4 rc=$?"
timeout 900 python tools/bench_configs.py --k4 > gpurun_out/c1/configs.jsonl 2> gpurun_out/c1/configs.err; echo "configs rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/c1/pytest.log
