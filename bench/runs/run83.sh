# two-phase: x segment cap around the default (4096) on c2 valued and pattern, c3 flickr
timeout 900 python bench/explore_pb.py c2 '[{"two_phase":1},{"two_phase":1,"pb_xcap":5120},{"two_phase":1,"pb_xcap":6144},{"two_phase":1,"pb_xcap":7168},{"two_phase":1,"pb_xcap":8192},{"two_phase":1,"pb_xcap":6144,"pb_group":5000000}]'
PATTERN=1 timeout 900 python bench/explore_pb.py c2 '[{"two_phase":1},{"two_phase":1,"pb_xcap":6144},{"two_phase":1,"pb_xcap":8192}]'
timeout 900 python bench/explore_pb.py c3_flickr '[{"two_phase":1},{"two_phase":1,"pb_xcap":6144},{"two_phase":1,"pb_xcap":8192}]'
