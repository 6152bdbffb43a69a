# knob sweep on the current box: L1 hot-column policy and L1-bypassing slot stream
L=$PWD/paper_1103_2405_b200/lib
O=gpurun_out/r65.jsonl; : > $O
python bench/explore_env.py c2 > /dev/null 2>&1
for lib in libtcspmv.so libtcspmv_streamna.so; do
  ENVS='[{}, {"TCSPMV_L1_HOT": 16384}, {"TCSPMV_L1_HOT": 49152}, {"TCSPMV_L1_HOT": 131072}, {"TCSPMV_CARVEOUT": 0}]' \
    TCSPMV_LIB=$L/$lib timeout 400 python bench/explore_env.py c2 >> $O 2>>gpurun_out/r65.err
done
