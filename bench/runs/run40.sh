# software pipelining of the slot stream: L1 prefetch of the next batch (pipe2) / register double buffer (pipe1)
L=$PWD/paper_1103_2405_b200/lib
O=gpurun_out/r40.jsonl; : > $O
export ENVS='[{}]'
python bench/explore_env.py c2 > /dev/null 2>&1
for lib in libtcspmv.so libtcspmv_pipe2.so libtcspmv_pipe2cm4.so libtcspmv_pipe1t768.so libtcspmv_pipe1t1024.so; do
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r40.err
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_env.py c2 --pattern >> $O 2>>gpurun_out/r40.err
  TCSPMV_LIB=$L/$lib timeout 300 python bench/explore_pr.py c2 2>>gpurun_out/r40.err | sed "s/^/{\"lib\": \"$lib\", \"pr\": /; s/$/}/" >> $O
done
