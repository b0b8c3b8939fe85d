A=paper_1503_02368_b200/lib/libeh_alt.so
for c in C3 C4 C2 C5; do
python tools/tri_sweep.py $c EH_DUMMY -
TRI_LIB=$A python tools/tri_sweep.py $c EH_DUMMY_NA -
done
