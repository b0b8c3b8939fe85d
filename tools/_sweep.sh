python tools/tri_sweep.py C5 EH_TEST_TRI_MID2 - 1024 1536 2048 4096 -
