# PDL chaining of standalone tile launches: default build vs TC_PDL=0; then the multi-tile parity tests
for L in libtcspmv.so libtcspmv_nopdl.so; do
  PDL_C4=1 TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pdl.py
done
timeout 600 python -m pytest tests/test_gpu_spmv.py -q -x 2>&1 | tail -2
