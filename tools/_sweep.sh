for c in C3 C4 C2 C5; do python tools/load_sweep.py $c EH_DUMMY - - ; done
EH_TIMING=1 python tools/profile_load.py --reps 3 2>&1 | grep timing | tail -1
python -m pytest tests -m gpu -x -q -k "bucket or dedup or batch" 2>&1 | tail -2
