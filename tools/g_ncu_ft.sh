#!/bin/bash
# ncu --set full (source counters) of the fused sweep kernels in one c3 step
O=gpurun_out; mkdir -p $O
export REXP_FUSE_FORCE=1 REXP_AUTOTUNE=0
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:'k_ft_' --launch-count 4 -o /tmp/ft_c3 -f python tools/profile_step.py --config c3_rsw_32x32_p16_x64 > $O/ft_ncu.log 2>&1
ncu -i /tmp/ft_c3.ncu-rep --page raw --csv > $O/ft_raw.csv 2>/dev/null
ncu -i /tmp/ft_c3.ncu-rep --page source --csv --print-source sass > $O/ft_source_sass.csv 2>/dev/null
ncu -i /tmp/ft_c3.ncu-rep --page source --csv --print-source cuda > $O/ft_source_cuda.csv 2>/dev/null
ncu -i /tmp/ft_c3.ncu-rep --page details > $O/ft_details.txt 2>/dev/null
tail -3 $O/ft_ncu.log; ls -la $O | grep ft_
