mkdir -p gpurun_out
O=gpurun_out/g2_err.txt; : > $O
timeout 300 python tools/c1_err.py default >> $O 2>&1
REXP_NO_SYM=1 timeout 300 python tools/c1_err.py nosym >> $O 2>&1
REXP_NO_XDIAG=1 timeout 300 python tools/c1_err.py noxdiag >> $O 2>&1
REXP_LEAF=dense timeout 300 python tools/c1_err.py leafdense >> $O 2>&1
REXP_LIB=librexp_cmul4.so timeout 300 python tools/c1_err.py cmul4 >> $O 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k shard > gpurun_out/g2_shard_tests.txt 2>&1
REXP_TIMING_DETAIL=1 timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/g2_c3_detail.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:'k_cgemm|k_leaf_gemm' --launch-count 40 -o /tmp/g2_c3 -f python tools/profile_step.py --config c3_rsw_32x32_p16_x64 > gpurun_out/g2_ncu.log 2>&1
ncu -i /tmp/g2_c3.ncu-rep --page raw --csv > gpurun_out/g2_c3_raw.csv 2>/dev/null
cp /tmp/g2_c3.ncu-rep gpurun_out/ 2>/dev/null
cat $O; grep -c . gpurun_out/g2_c3_raw.csv
