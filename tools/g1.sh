mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -k "not c3_sampled and not shard_pole_sums" --durations=15 > gpurun_out/g1_tests.txt 2>&1
timeout 600 python bench.py > gpurun_out/g1_bench_c3.log 2>&1
timeout 300 python bench.py --config c1_rsw_16x16_p16 --no-cpu-baseline > gpurun_out/g1_bench_c1.log 2>&1
tail -25 gpurun_out/g1_tests.txt; tail -1 gpurun_out/g1_bench_c3.log | cut -c1-300; tail -1 gpurun_out/g1_bench_c1.log | cut -c1-300
