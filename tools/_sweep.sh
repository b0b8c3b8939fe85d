A=paper_1503_02368_b200/lib/libeh_alt.so
for c in C5 C3 C4 C2; do
python tools/tri_sweep.py $c EH_DUMMY -
TRI_LIB=$A python tools/tri_sweep.py $c EH_DUMMY_PACKED -
done
