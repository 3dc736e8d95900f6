#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "symmetric_pair" 2>&1 | tail -3 > $O/x1_tests.txt
cat $O/x1_tests.txt
timeout 600 python bench.py --steps 20 --no-cpu-baseline > $O/x1_bench_c3.log 2>&1
tail -1 $O/x1_bench_c3.log | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['impl_details']['merge_kernels'])
print({k: v['ms_per_step'] for k, v in d['roofline']['per_class'].items()})
"
