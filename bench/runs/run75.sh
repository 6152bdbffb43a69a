for L in libtcspmv.so libtcspmv_f10.so libtcspmv_f11.so; do
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L VARIANTS='[]' timeout 300 python bench/explore_solver_plan.py c2 2>&1 | sed "s/^/$L /"
done
