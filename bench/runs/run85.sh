# two-phase pipeline depth: 3 stages per CTA with smaller items (2 CTAs per SM) vs the 2-stage default
V='[{"two_phase":1},{"two_phase":1,"pb_chunk":2048,"pb_xcap":3072,"pb_region":4096},{"two_phase":1,"pb_chunk":2560,"pb_xcap":3072,"pb_region":4096},{"two_phase":1,"pb_chunk":3072,"pb_xcap":3072,"pb_region":4096}]'
timeout 900 python bench/explore_pb.py c2 "$V"
TCSPMV_LIB=$PWD/paper_1103_2405_b200/lib/libtcspmv_st3.so timeout 900 python bench/explore_pb.py c2 "$V"
