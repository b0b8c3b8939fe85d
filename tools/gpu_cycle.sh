#!/bin/bash
# One GPU iteration (run under gpurun): parity tests, bench, optional ncu capture.
#   tools/gpu_cycle.sh [tests|notests] [ncu-regex|none] [extra pytest -k expr]
mkdir -p gpurun_out
T=${1:-tests}; NCU=${2:-none}; K=${3:-}
if [ "$T" = "tests" ]; then
  if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 -k "$K" > gpurun_out/pytest_gpu.log 2>&1
  else timeout 1500 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/pytest_gpu.log 2>&1; fi
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -4 gpurun_out/pytest_gpu.log
fi
EH_TIMING=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
grep "eh timing" gpurun_out/bench.log | tail -1
grep '^{' gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','count_ms','load_ms','triangles']}, d['roofline']['frac'], d['e2e']['value'])"
if [ "$NCU" != "none" ]; then
  timeout 300 python tools/profile_count.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU -s 1 -c 1 -o gpurun_out/prof python tools/profile_count.py --reps 2 > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"; cat gpurun_out/prof_plain.log | head -3
fi
