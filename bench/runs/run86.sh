# two-phase: L2 prefetch of the streams of the item 1 / 2 / 3 claims ahead (PB_PF_AHEAD) vs none
for L in libtcspmv_pf0.so libtcspmv.so libtcspmv_pf2.so libtcspmv_pf3.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 900 python bench/explore_pb.py c2 '[{"two_phase":1}]' | grep variant
  PATTERN=1 TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 900 python bench/explore_pb.py c2 '[{"two_phase":1}]' | grep variant
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 900 python bench/explore_pb.py c3_flickr '[{"two_phase":1}]' | grep variant
done
