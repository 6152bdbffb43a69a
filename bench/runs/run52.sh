# occupancy variants of the tile kernel: 48 / 64 warps per SM (register caps 40 / 32, with spills)
L=$PWD/paper_1103_2405_b200/lib
O=gpurun_out/r52.jsonl; : > $O
python bench/explore_env.py c2 > /dev/null 2>&1
for lib in libtcspmv.so libtcspmv_minb3.so libtcspmv_minb3cm1.so libtcspmv_minb4.so; do
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r52.err
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 --pattern >> $O 2>>gpurun_out/r52.err
done
