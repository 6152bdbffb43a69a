# hub columns in shared memory: 2 x 512-thread CTAs (prefix duplicated per CTA) vs one 1024-thread CTA per SM
L=$PWD/paper_1103_2405_b200/lib
O=gpurun_out/r42.jsonl; : > $O
python bench/explore_env.py c2 > /dev/null 2>&1
for lib in libtcspmv.so libtcspmv_t1024.so; do
  for pat in "" "--pattern"; do
    ENVS='[{}, {"TCSPMV_PREFIX": 16384}, {"TCSPMV_PREFIX": 24576}, {"TCSPMV_PREFIX": 40960}, {"TCSPMV_PREFIX": 49152}, {"TCSPMV_PREFIX": 55296}, {}]' \
      TCSPMV_LIB=$L/$lib timeout 400 python bench/explore_env.py c2 $pat >> $O 2>>gpurun_out/r42.err
  done
done
for lib in libtcspmv.so libtcspmv_t1024.so; do
  for pf in 0 49152; do
    TCSPMV_PREFIX=$pf TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_pr.py c2 2>>gpurun_out/r42.err | sed "s/^/{\"lib\": \"$lib\", \"prefix\": $pf, \"pr\": /; s/$/}/" >> $O
  done
done
