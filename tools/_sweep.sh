for c in C3 C4 C2; do
python tools/load_sweep.py $c EH_TEST_BKT_PART_MATCH - 1
done
EH_TIMING=1 python tools/profile_load.py --reps 3 2>&1 | grep timing | tail -1
EH_TIMING=1 python tools/profile_load.py --config C5 --reps 2 2>&1 | grep timing | tail -1
