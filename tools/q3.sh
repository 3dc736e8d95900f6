# parity after a kernel change + c3 / c1 bench lines
mkdir -p gpurun_out
R=${1:-q3}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "not c1 and not sampled_rhs and not shard_pole" 2>&1 | tail -15 > gpurun_out/${R}_tests.txt
timeout 300 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/${R}_bench_c3.log 2>&1
timeout 200 python bench.py --config c1_rsw_16x16_p16 --steps 50 --no-cpu-baseline > gpurun_out/${R}_bench_c1.log 2>&1
cat gpurun_out/${R}_tests.txt
for f in c3 c1; do python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/${R}_bench_$f.log").read().splitlines() if l.startswith("{")][-1])
print("$f", round(d["value"]/1e6,2), "M dof-steps/s", round(d["ms_per_step"],3), "ms", {k: v["ms_per_step"] for k, v in d["roofline"]["per_class"].items()})
PY
done
if [ "${NCU:-0}" = "1" ]; then
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:'k_cgemm|k_leaf_gemm|k_upx|k_root' --launch-count 40 \
    -o /tmp/${R}_c3_full -f python tools/profile_step.py --config c3_rsw_32x32_p16_x64 > gpurun_out/${R}_ncu_full.log 2>&1
ncu -i /tmp/${R}_c3_full.ncu-rep --page raw --csv > gpurun_out/${R}_c3_raw.csv 2>/dev/null
ncu -i /tmp/${R}_c3_full.ncu-rep --page details --csv > gpurun_out/${R}_c3_details.csv 2>/dev/null
ls -la gpurun_out | tail -5
fi
