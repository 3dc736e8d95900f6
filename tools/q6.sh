mkdir -p gpurun_out
R=${1:-q6}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config0" 2>&1 | tail -3 > gpurun_out/${R}_tests.txt
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/${R}_bench_c3.log 2>&1
cat gpurun_out/${R}_tests.txt
python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/${R}_bench_c3.log").read().splitlines() if l.startswith("{")][-1])
print("c3", round(d["value"]/1e6,2), "M", round(d["ms_per_step"],2), "ms", {k: v["ms_per_step"] for k, v in d["roofline"]["per_class"].items()})
print(d["impl_details"]["merge_kernels"])
PY
