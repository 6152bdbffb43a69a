# PDL trigger at kernel start (default build) vs at the end of the CTA's workloads vs no PDL, twice each
for r in 1 2; do
for L in libtcspmv.so libtcspmv_pdllate.so libtcspmv_nopdl.so; do
  PDL_C4=$([ $r = 1 ] && echo 1) TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pdl.py
done
done
