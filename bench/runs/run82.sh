# two-phase parameter sweep on c2 valued (rcap / ccap / xcap / group)
timeout 1500 python bench/explore_pb.py c2 '[{"two_phase":1},
 {"two_phase":1,"pb_region":4096},{"two_phase":1,"pb_region":8192},
 {"two_phase":1,"pb_chunk":3072},{"two_phase":1,"pb_chunk":5120},
 {"two_phase":1,"pb_xcap":2048},{"two_phase":1,"pb_xcap":6144},
 {"two_phase":1,"pb_group":3000000},{"two_phase":1,"pb_group":8000000},{"two_phase":1,"pb_group":12000000},
 {"two_phase":1,"pb_chunk":3072,"pb_region":4096},{"two_phase":1,"pb_chunk":5120,"pb_xcap":6144}]'
