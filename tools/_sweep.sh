for c in C3 C4 C2 C5; do python tools/tri_sweep.py $c EH_DUMMY - ; done
for c in C3 C4 C2; do WHAT=k4 KNOB=bin_thread_max python tools/bin_sweep.py $c 8 16; WHAT=pv KNOB=bin_thread_max python tools/bin_sweep.py $c 8 16; done
python -m pytest tests -m gpu -x -q -k "thread or binning or invariance or configs" 2>&1 | tail -2
