#!/bin/bash
# second reflection (sym2): parity of every R2 >= 16 path, then the c3 bench line with and without it
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric_pair or many_rhs or fused" 2>&1 | tail -4 > $O/s2_tests.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "64rhs" 2>&1 | grep -E "rel L2|passed|failed" | cut -c1-200 >> $O/s2_tests.txt
cat $O/s2_tests.txt
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/s2_bench_c3.log 2>&1
timeout 600 env REXP_NO_SYM2=1 python bench.py --steps 20 --no-cpu-baseline > $O/s2_bench_c3_off.log 2>&1
for f in $O/s2_bench_c3.log $O/s2_bench_c3_off.log; do echo $f; tail -1 $f | python -c "
import sys, json
try:
    d = json.loads(sys.stdin.read())
    print(d['value'], d['ms_per_step'], d['impl_details']['merge_kernels'][-260:])
    print({k: v['ms_per_step'] for k, v in d['roofline']['per_class'].items()}, d['roofline']['whole_step'])
except Exception as e:
    print('ERR', e)
"; done
