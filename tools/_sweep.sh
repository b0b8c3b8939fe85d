A=paper_1503_02368_b200/lib/libeh_alt.so
export TRI_QUERY=k4
for c in C4 C3 C2; do
python tools/tri_sweep.py $c EH_DUMMY_VEC -
TRI_LIB=$A python tools/tri_sweep.py $c EH_DUMMY_SCALAR -
done
python tools/tri_sweep.py C4 EH_DUMMY_VEC -
python -m pytest tests -m gpu -x -q -k "k4 or 4clique or K4 or cliques" 2>&1 | tail -2
