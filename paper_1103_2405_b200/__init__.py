"""paper_1103_2405_b200 -- B200-native tiled-composite SpMV and the PageRank / HITS / RWR power
iterations on it (Yang, Parthasarathy & Sadayappan, VLDB 2011).  The compute path is the C-ABI
library lib/libtcspmv.so (include/spmv.h); this package only marshals arguments."""
from .api import (Comm, Plan, Solver, bitonic_partition, needed_lists, hits, iter_opts, make_options, pagerank,
                  partition_plan, rwr)
from ._capi import LIB_PATH, SpmvError, lib

__all__ = ["Plan", "Solver", "Comm", "pagerank", "hits", "rwr", "bitonic_partition", "partition_plan", "needed_lists",
           "make_options", "iter_opts", "SpmvError", "lib", "LIB_PATH"]
