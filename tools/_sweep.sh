A=paper_1503_02368_b200/lib/libeh_alt.so
for c in C3 C4 C2 C5; do
python tools/pv_sweep.py $c 0,0
TRI_LIB=$A python tools/pv_sweep.py $c 0,0 | sed 's/$/ (no filter)/'
done
python -m pytest tests -m gpu -x -q -k "next1" 2>&1 | tail -2
