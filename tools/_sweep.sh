for sh in 0 -1; do
EH_TEST_BKT_SHIFT=$sh EH_TIMING=1 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "eh timing|^\{" | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print({k:round(d[k],3) for k in ['ms_per_step','count_ms','load_ms']})
    else: print(l.strip()[100:230])
"
done
python tools/load_sweep.py C4 EH_TEST_BKT_SHIFT 0
python tools/load_sweep.py C2 EH_TEST_BKT_SHIFT 0
