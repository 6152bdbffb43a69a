# PDL with the plan's rule (short launches only) vs TC_PDL off; SpMV and solver parity tests
for L in libtcspmv.so libtcspmv_nopdl.so; do
  PDL_C4=1 TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pdl.py
done
timeout 900 python -m pytest tests/test_gpu_spmv.py tests/test_gpu_iter.py -q -x -k "not c4" 2>&1 | tail -2
