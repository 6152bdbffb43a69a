# Which L1TEX sub-unit binds the tile kernel?  breakdown of l1tex__throughput for: default,
# t1024 + smem prefix 32K, bulk-copy stream kernel.  Plus host RAM of the box (c4 planning).
free -g > gpurun_out/r37_free.txt; nproc >> gpurun_out/r37_free.txt
L=$PWD/paper_1103_2405_b200/lib
M="breakdown:l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.sum"
run() { tag=$1; shift; env "$@" ENVS='[{}]' timeout 600 ncu --metrics $M --clock-control none -k regex:tc_spmv -s 5 -c 1 --csv --print-units base \
   python bench/explore_env.py c2 > gpurun_out/r37_$tag.csv 2>&1; }
python bench/explore_env.py c2 > /dev/null 2>&1   # cache the graph
run base TCSPMV_LIB=$L/libtcspmv.so
run pre32k TCSPMV_LIB=$L/libtcspmv_t1024.so TCSPMV_PREFIX=32768
run stream TCSPMV_LIB=$L/libtcspmv.so TCSPMV_KERNEL=stream
ENVS="[{}]" TCSPMV_LIB=$L/libtcspmv.so timeout 600 ncu --metrics $M --clock-control none -k regex:tc_spmv -s 5 -c 1 --csv --print-units base python bench/explore_env.py c2 --pattern > gpurun_out/r37_pattern.csv 2>&1
