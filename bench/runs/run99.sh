# batched RWR after the unconditional loads: x-row loads in flight per warp step (TC_BATCH_U; default 16)
for L in libtcspmv_u8.so libtcspmv_u12.so libtcspmv.so libtcspmv_u24.so libtcspmv_u32.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_batch_wl.py 2>&1 | grep -E '"wl": (512|1024|2048)'
done
