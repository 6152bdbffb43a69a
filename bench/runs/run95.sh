# one-pass SpMV (EpiStore): FLAG_ACC check only in launches that can hold accumulating rows vs before
for r in 1 2; do
for L in libtcspmv_prev.so libtcspmv.so; do
  echo "lib $L"
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c2 '[{"two_phase":0},{"two_phase":0,"num_tiles":2,"tile_width":49152}]' | grep variant
  TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/$L timeout 600 python bench/explore_pb.py c3_flickr '[{"two_phase":0}]' | grep variant
done
done
PDL_C4=1 timeout 900 python bench/explore_pdl.py 2>&1 | grep c4
PDL_C4=1 TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/libtcspmv_prev.so timeout 900 python bench/explore_pdl.py 2>&1 | grep c4
