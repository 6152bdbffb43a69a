# L1 / shared-memory x-residency experiments on c2 (stream no-allocate, hot-column L1 priority, prefix in smem)
L=$PWD/paper_1103_2405_b200/lib
O=gpurun_out/r36.jsonl; : > $O
export ENVS='[{}, {"TCSPMV_L1_HOT": 32768}, {"TCSPMV_L1_HOT": 65536}, {"TCSPMV_PREFIX": 16384}]'
for lib in libtcspmv.so libtcspmv_na.so libtcspmv_m3.so; do
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r36.err
done
export ENVS='[{}, {"TCSPMV_PREFIX": 16384}, {"TCSPMV_PREFIX": 32768}, {"TCSPMV_PREFIX": 49152}, {"TCSPMV_PREFIX": 53248}, {"TCSPMV_PREFIX": 49152, "TCSPMV_L1_HOT": 65536}]'
for lib in libtcspmv_t1024.so libtcspmv_t1024na.so; do
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r36.err
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 --pattern >> $O 2>>gpurun_out/r36.err
done
