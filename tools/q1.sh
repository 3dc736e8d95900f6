mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "c2r or live_oracle" 2>&1 | tail -15 > gpurun_out/q1_tests.txt
timeout 400 python bench.py --steps 20 > gpurun_out/q1_bench_c3.log 2>&1
timeout 900 python bench.py --config c2_wave_32x32_p16 --shard auto --steps 5 --no-cpu-baseline > gpurun_out/q1_bench_c2s.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/q1_fp64_peak.txt 2>&1
cat gpurun_out/q1_tests.txt; tail -c 300 gpurun_out/q1_bench_c3.log; tail -c 1500 gpurun_out/q1_bench_c2s.log
