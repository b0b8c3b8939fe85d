P=paper_1503_02368_b200/lib
python tools/tri_sweep.py C5 EH_DUMMY -
for v in cg4 nw8 nw8cg4 tab4096 nw2; do
TRI_LIB=$P/libeh_$v.so python tools/tri_sweep.py C5 EH_DUMMY_$v -
done
python tools/tri_sweep.py C5 EH_DUMMY -
