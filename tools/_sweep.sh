for c in C3 C4; do
python tools/tri_sweep.py $c EH_TEST_TRI_CARVEOUT_W - 60 50 40
python tools/tri_sweep.py $c EH_TEST_TRI_CARVEOUT_T - 60 50 30
python tools/tri_sweep.py $c EH_TEST_TRI_CARVEOUT_C - 55 60 65 70
done
