# source-level stalls of the one-pass tile kernel in the HITS iteration after prefetch_rm (c2)
R=r02e
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_spmv_tile -s 2 -c 1 -o gpurun_out/${R}_h \
    python -c "
import sys; sys.path.insert(0,'.')
import graphgen; from paper_1103_2405_b200 import Solver
G=graphgen.make_graph('c2'); s=Solver('hits',G.n,G.row_ptr,G.col,device=0,iter_kw=dict(fixed_iters=4,host_loop=1)); print(s.run())
" > gpurun_out/${R}_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/${R}_h.ncu-rep --page source --csv --print-units base > gpurun_out/${R}_src.csv 2>&1
ncu -i gpurun_out/${R}_h.ncu-rep --page raw --csv --print-units base > gpurun_out/${R}_raw.csv 2>&1
rm -f gpurun_out/${R}_h.ncu-rep
