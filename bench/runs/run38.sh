L=$PWD/paper_1103_2405_b200/lib
M="breakdown:l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"
run() { tag=$1; shift; env "$@" ENVS='[{}]' timeout 600 ncu --metrics $M --clock-control none -k regex:tc_spmv -s 5 -c 1 --csv --print-units base \
   python bench/explore_env.py c2 > gpurun_out/r38_$tag.csv 2>&1; }
python bench/explore_env.py c2 > /dev/null 2>&1   # cache the graph
run base TCSPMV_LIB=$L/libtcspmv.so
run na TCSPMV_LIB=$L/libtcspmv_na.so
run pre32k TCSPMV_LIB=$L/libtcspmv_t1024.so TCSPMV_PREFIX=32768
run pre48k TCSPMV_LIB=$L/libtcspmv_t1024na.so TCSPMV_PREFIX=49152
run hot TCSPMV_LIB=$L/libtcspmv_na.so TCSPMV_L1_HOT=49152
