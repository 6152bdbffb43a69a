# default x segment cap 6144 (with the two-CTA fallback): c1-c4 two-phase timings and parity tests
timeout 900 python bench/explore_pb.py c2 '[{"two_phase":1},{"two_phase":1,"pb_xcap":4096},{}]'
PATTERN=1 timeout 900 python bench/explore_pb.py c2 '[{"two_phase":1},{"two_phase":1,"pb_xcap":4096}]'
timeout 900 python bench/explore_pb.py c3_flickr '[{"two_phase":1},{"two_phase":1,"pb_xcap":4096},{}]'
timeout 900 python bench/explore_pb.py c3_youtube '[{"two_phase":1},{"two_phase":1,"pb_xcap":4096},{}]'
timeout 900 python bench/explore_pb.py c1 '[{"two_phase":1},{"two_phase":1,"pb_xcap":4096},{}]'
timeout 1200 python -m pytest tests/test_two_phase.py tests/test_gpu_spmv.py -q -x 2>&1 | tail -2
