# CTA size 256 x 4 per SM vs 512 x 2 (same 32 warps per SM)
L=$PWD/paper_1103_2405_b200/lib
O=gpurun_out/r71.jsonl; : > $O
python bench/explore_env.py c2 > /dev/null 2>&1
for lib in libtcspmv.so libtcspmv_t256.so libtcspmv.so libtcspmv_t256.so; do
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r71.err
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 --pattern >> $O 2>>gpurun_out/r71.err
done
