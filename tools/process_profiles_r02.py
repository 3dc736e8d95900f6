"""Turn the raw outputs of tools/round_measure_r02.sh (gpurun_out/) into the
committed summaries under profiles/:

  profiles/<R>_bench_<cfg>.json          bench JSON lines (c3 headline, c1, c2r, c2/c4 shards, reference arm)
  profiles/<R>_gpu_tests.txt             pytest -m gpu summary
  profiles/<R>_launches_<c>.csv          ncu launch list of the bench's timed region (time + DRAM bytes per launch)
  profiles/<R>_launch_shares_<c>.txt     per-kernel and per-class shares of that list
  profiles/<R>_c3_ncu_details.txt        ncu --set full of the top kernels of one c3 step
  profiles/traffic.json                  DRAM bytes per launch, keyed "workload/class" (bench.py roofline.traffic)

    python tools/process_profiles_r02.py r02
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
WORKLOAD = {"c3": "c3_rsw_32x32_p16_x64", "c1": "c1_rsw_16x16_p16"}
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}

# kernel name -> bench class (api.KERNEL_CLASSES)
def klass(name, grid):
    if "k_spec_pre" in name or "k_pre" in name:
        return "pre"
    if "k_leaf_gemm_up" in name or "k_leaf_up" in name:
        return "leaf_up"
    if "k_leaf_gemm_down" in name or "k_leaf_down" in name:
        return "leaf_down"
    if "k_root" in name:
        return "root"
    if "k_spec_back" in name or "k_pole_sum" in name:
        return "pole_sum"
    if "k_recover" in name:
        return "recover"
    return "merge"


def last_json_line(path):
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.startswith("{")]
    return lines[-1] if lines else None


def launches(r, c):
    path = os.path.join(RAW, f"{r}_launches_{c}.csv")
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    hi = [i for i, row in enumerate(rows) if "Kernel Name" in row][0]
    h = rows[hi]
    idx = {k: i for i, k in enumerate(h)}
    per = collections.OrderedDict()
    for row in rows[hi + 1:]:
        if len(row) != len(h):
            continue
        key = (row[idx["ID"]], row[idx["Kernel Name"]], row[idx["Grid Size"]], row[idx["Block Size"]])
        per.setdefault(key, {})[row[idx["Metric Name"]]] = float(row[idx["Metric Value"]]) * MULT.get(
            row[idx["Metric Unit"]], 1.0)
    out = []
    for (i, name, grid, block), m in per.items():
        out.append((i, name.replace("void ", "").replace("rexp::dev::", ""), grid, block,
                    m.get("gpu__time_duration.sum", 0.0) * 1e6,
                    m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)))
    with open(os.path.join(OUT, f"{r}_launches_{c}.csv"), "w") as f:
        f.write("# ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                "dram__bytes_write.sum --clock-control none --csv\n")
        f.write(f"#   python bench.py --config {WORKLOAD[c]} --steps 1 --warmup 3 --no-cpu-baseline  (the bench's\n")
        f.write("#   timed region: one step, CUDA-graph replay).  Per-launch times are cold-cache and serialised:\n")
        f.write("#   compare SHARES, not absolute values.\n")
        f.write("id,kernel,grid,block,us,dram_bytes\n")
        for o in out:
            f.write(f'{o[0]},"{o[1]}","{o[2]}","{o[3]}",{o[4]:.2f},{o[5]:.0f}\n')
    tot = sum(o[4] for o in out)
    cls = collections.OrderedDict()
    kern = collections.OrderedDict()
    traffic = collections.defaultdict(list)
    down = False
    for o in out:
        short = o[1].split("(")[0]
        base = short.split("<")[0]
        kl = klass(base, o[2])
        # launch order of a pole chunk: leaf up, merges up, root, merges down, leaf down
        if kl == "root":
            down = True
        elif kl in ("leaf_up", "pre"):
            down = False
        if kl == "merge":
            kl = "merge_down" if down else "merge_up"
        cls.setdefault(kl, [0.0, 0, 0.0])
        cls[kl][0] += o[4]; cls[kl][1] += 1; cls[kl][2] += o[5]
        kern.setdefault(base, [0.0, 0])
        kern[base][0] += o[4]; kern[base][1] += 1
        traffic[kl].append(o[5])
    lines = [f"# {len(out)} launches, {tot:.1f} us serialised (ncu, cold)", "# class: us, share, launches, DRAM GB"]
    for k, v in cls.items():
        lines.append(f"{k:12s} {v[0]:10.1f} us {100 * v[0] / tot:5.1f}%  {v[1]:4d} launches  {v[2] / 1e9:8.3f} GB")
    lines.append("# kernel: us, share, launches")
    for k, v in kern.items():
        lines.append(f"{k:22s} {v[0]:10.1f} us {100 * v[0] / tot:5.1f}%  {v[1]:4d}")
    open(os.path.join(OUT, f"{r}_launch_shares_{c}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return {f"{WORKLOAD[c]}/{k}": int(sum(v) / len(v)) for k, v in traffic.items()}


def full_details(r):
    path = os.path.join(RAW, f"{r}_c3_raw.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path).read().splitlines()))
    h, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(h)}

    def val(row, k, default=0.0):
        try:
            return float(row[idx[k]])
        except (KeyError, ValueError):
            return default

    stall = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
             k.endswith("_per_issue_active.ratio")]
    dm = "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"
    lines = ["# ncu --set full --clock-control none -k regex:'k_cgemm|k_leaf_gemm|k_upx|k_root|k_spec|k_recover' --launch-count 40",
             "#   python tools/profile_step.py --config c3_rsw_32x32_p16_x64   (one warm c3 step, first pole chunk)",
             "# columns: grid | time | DRAM GB, TB/s | warps active % | regs | DMMA-pipe % | FP64-pipe % | top stalls", ""]
    seen = set()
    for row in rows[2:]:
        name = row[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("rexp::dev::", "")
        key = (name, row[idx["Grid Size"]])
        if key in seen:
            continue
        seen.add(key)
        t = val(row, "gpu__time_duration.sum") * MULT.get(units[idx["gpu__time_duration.sum"]], 1.0)
        gb = (val(row, "dram__bytes_read.sum") * MULT.get(units[idx["dram__bytes_read.sum"]], 1) +
              val(row, "dram__bytes_write.sum") * MULT.get(units[idx["dram__bytes_write.sum"]], 1)) / 1e9
        st = sorted(((val(row, k), k.replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for k in stall), reverse=True)[:3]
        lines.append(f"{name:44s} {row[idx['Grid Size']]:>14s} {t * 1e3:8.3f} ms {gb:7.3f} GB "
                     f"{gb / t / 1e3 if t else 0:5.2f} TB/s warps {val(row, 'sm__warps_active.avg.pct_of_peak_sustained_active'):3.0f}% "
                     f"regs {val(row, 'launch__registers_per_thread'):3.0f} dmma {val(row, dm):4.1f}% "
                     f"fp64 {val(row, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):4.1f}% | "
                     + ", ".join(f"{n} {v:.1f}" for v, n in st))
    open(os.path.join(OUT, f"{r}_c3_ncu_details.txt"), "w").write("\n".join(lines) + "\n")


def main():
    r = sys.argv[1] if len(sys.argv) > 1 else "r02"
    for src in ("c3", "c1", "c2r", "reference", "c2_shard", "c4_shard"):
        p = os.path.join(RAW, f"{r}_bench_{src}.log")
        if os.path.exists(p):
            ln = last_json_line(p)
            if ln:
                open(os.path.join(OUT, f"{r}_bench_{src}.json"), "w").write(ln + "\n")
    t = os.path.join(RAW, f"{r}_gpu_tests.txt")
    if os.path.exists(t):
        open(os.path.join(OUT, f"{r}_gpu_tests.txt"), "w").write(open(t).read())
    traffic = {}
    for c in ("c3", "c1"):
        tr = launches(r, c)
        if tr:
            traffic.update(tr)
    if traffic:
        traffic["_about"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes; mean over the class's "
                             f"launches in one bench step), from profiles/{r}_launches_<c>.csv")
        json.dump(traffic, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)
    full_details(r)


if __name__ == "__main__":
    main()
