#!/bin/bash
# c1 accuracy study: one to three c1 steps against the oracle golden under kernel variants
mkdir -p gpurun_out
O=gpurun_out/g_err.txt; : > $O
timeout 300 python tools/c1_err.py default >> $O 2>&1
REXP_NO_SYM=1 timeout 300 python tools/c1_err.py nosym >> $O 2>&1
REXP_NO_XDIAG=1 timeout 300 python tools/c1_err.py noxdiag >> $O 2>&1
REXP_LEAF=dense timeout 300 python tools/c1_err.py leafdense >> $O 2>&1
REXP_LIB=librexp_cmul4.so timeout 300 python tools/c1_err.py cmul4 >> $O 2>&1
REXP_LANES=1 timeout 300 python tools/c1_err.py lanes1 >> $O 2>&1
REXP_AUTOTUNE=0 timeout 300 python tools/c1_err.py notune >> $O 2>&1
cat $O
