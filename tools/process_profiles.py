"""Turn the raw outputs of tools/round_measure.sh (gpurun_out/) into the
committed summaries under profiles/:

  profiles/<R>_bench_{c1,c3,c2r_wave,reference}.json   bench JSON lines
  profiles/<R>_gpu_tests.txt                            pytest -m gpu summary
  profiles/<R>_launches.csv                             ncu launch list of the bench's timed region
  profiles/<R>_leaf_ncu_details.txt                     ncu --set full of the spectral leaf kernels
  profiles/<R>_merge_ncu_details.txt                    ncu --set full of the first 24 merge launches of a step
  profiles/traffic.json                                 dram bytes per launch (bench.py roofline.traffic)

    python tools/process_profiles.py r01
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")


def last_json_line(path):
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.startswith("{")]
    return lines[-1]


def launches(r):
    rows = list(csv.reader(open(os.path.join(RAW, f"{r}_launches.csv"))))
    hi = [i for i, row in enumerate(rows) if "Kernel Name" in row][0]
    h = rows[hi]
    idx = {k: i for i, k in enumerate(h)}
    out = [(row[idx["ID"]], row[idx["Kernel Name"]], row[idx["Grid Size"]], row[idx["Block Size"]],
            float(row[idx["Metric Value"]]) / 1e3) for row in rows[hi + 1:] if len(row) == len(h)]
    with open(os.path.join(OUT, f"{r}_launches.csv"), "w") as f:
        f.write("# ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv\n")
        f.write("#   python bench.py --steps 2 --warmup 3 --no-cpu-baseline   (the bench's timed region only:\n")
        f.write("#   2 steps of c1, CUDA-graph replay, 2 pole lanes -> every stage appears once per lane)\n")
        f.write("# per-launch times are cold-cache and serialised: compare SHARES, not absolute values\n")
        f.write("id,kernel,grid,block,us\n")
        for o in out:
            f.write(f'{o[0]},"{o[1]}","{o[2]}","{o[3]}",{o[4]:.2f}\n')
    tot = sum(o[4] for o in out)
    cls = collections.OrderedDict()
    for o in out:
        k = o[1].split("(")[0].split("<")[0].replace("void ", "")
        cls[k] = cls.get(k, 0.0) + o[4]
    print(f"{len(out)} launches, {tot:.1f} us")
    for k, v in cls.items():
        print(f"  {k:20s} {v:9.1f} us {100 * v / tot:5.1f}%")


def leaf_ncu(r):
    rep = os.path.join(RAW, f"{r}_leaf_full.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(h)}
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.avg.per_cycle_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
    stall = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
             k.endswith("_per_issue_active.ratio")]
    lines = ["# ncu --set full --clock-control none --import-source on -k regex:k_leaf_spec",
             "#   python tools/profile_step.py   (one warm step of c1_rsw_16x16_p16: 282 half poles in 2 lanes,",
             "#   256 leaves, R2 = 2; the capture lists each lane's launch)", ""]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = {}
    for row in rows[2:]:
        name = row[idx["Kernel Name"]].split("(")[0]
        lines.append(f"== {name}  grid {row[idx['Grid Size']]} block {row[idx['Block Size']]}")
        for w in want:
            if w in idx:
                lines.append(f"  {w:62s} {row[idx[w]]:>16s} {units[idx[w]]}")
        st = sorted(((float(row[idx[k]] or 0), k.replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for k in stall), reverse=True)[:6]
        lines.append("  top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st))
        lines.append("")
        tb = (float(row[idx["dram__bytes_read.sum"]]) * mult[units[idx["dram__bytes_read.sum"]]] +
              float(row[idx["dram__bytes_write.sum"]]) * mult[units[idx["dram__bytes_write.sum"]]])
        traffic.setdefault("leaf_up" if "up" in name else "leaf_down", []).append(tb)
    with open(os.path.join(OUT, f"{r}_leaf_ncu_details.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    t = {k: int(sum(v) / len(v)) for k, v in traffic.items()}
    t["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes; mean over the lane "
                   "launches), ncu --set full --clock-control none of tools/profile_step.py (one warm c1 "
                   f"step); see profiles/{r}_leaf_ncu_details.txt")
    json.dump(t, open(os.path.join(OUT, "traffic.json"), "w"), indent=1)


def merge_ncu(r):
    """profiles/<R>_merge_ncu_details.txt: one line per captured merge launch."""
    path = os.path.join(RAW, f"{r}_merge_raw.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path).read().splitlines()))
    h, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(h)}
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tmult = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    stall = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
             k.endswith("_per_issue_active.ratio")]
    dmma = [k for k in h if "dmma" in k and k.endswith("pct_of_peak_sustained_active")]

    def val(row, k, default=0.0):
        try:
            return float(row[idx[k]])
        except (KeyError, ValueError):
            return default

    def count(row, k):
        u = units[idx[k]] if k in idx else ""
        return val(row, k) * (1e3 if u.startswith("K") else 1e6 if u.startswith("M") else 1.0)

    def spr(row, op):   # L1 sectors per global request
        req = count(row, f"l1tex__t_requests_pipe_lsu_mem_global_op_{op}.sum")
        return count(row, f"l1tex__t_sectors_pipe_lsu_mem_global_op_{op}.sum") / req if req else 0.0

    lines = ["# ncu --set full --clock-control none -k regex:'k_cgemm|k_gemv_sym' --launch-count 24",
             "#   python tools/profile_step.py   (one warm c1 step: the first 24 merge launches of the step,",
             "#   2 pole lanes of 141 half poles; cold, serialised per-launch numbers)",
             "# columns: us | DRAM read+write MB, TB/s | warps active % | regs | FP64-pipe % | "
             + ("DMMA-pipe % | " if dmma else "") + "L1 global ld/st sectors per request | top stalls", ""]
    for row in rows[2:]:
        name = row[idx["Kernel Name"]].split("(")[0].replace("void ", "").replace("rexp::dev::", "")
        us = val(row, "gpu__time_duration.sum") * tmult.get(units[idx["gpu__time_duration.sum"]], 1.0)
        mb = (val(row, "dram__bytes_read.sum") * mult.get(units[idx["dram__bytes_read.sum"]], 1) +
              val(row, "dram__bytes_write.sum") * mult.get(units[idx["dram__bytes_write.sum"]], 1)) / 1e6
        st = sorted(((val(row, k), k.replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for k in stall), reverse=True)[:3]
        dm = f"dmma {max(val(row, k) for k in dmma):4.1f}% " if dmma else ""
        lines.append(
            f"{name:46s} {row[idx['Grid Size']]:>13s} {us:7.1f} us {mb:7.1f} MB {mb / us if us else 0.0:4.2f} TB/s "
            f"warps {val(row, 'sm__warps_active.avg.pct_of_peak_sustained_active'):3.0f}% "
            f"regs {val(row, 'launch__registers_per_thread'):3.0f} "
            f"fp64 {val(row, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):4.1f}% {dm}"
            f"ld {spr(row, 'ld'):4.1f} st {spr(row, 'st'):4.1f} | "
            + ", ".join(f"{n} {v:.1f}" for v, n in st))
    with open(os.path.join(OUT, f"{r}_merge_ncu_details.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


def main():
    r = sys.argv[1] if len(sys.argv) > 1 else "r01"
    for src, dst in (("c1", "c1"), ("c3", "c3"), ("c2r", "c2r_wave"), ("reference", "reference")):
        p = os.path.join(RAW, f"{r}_bench_{src}.log")
        if os.path.exists(p):
            open(os.path.join(OUT, f"{r}_bench_{dst}.json"), "w").write(last_json_line(p) + "\n")
    t = os.path.join(RAW, f"{r}_gpu_tests.txt")
    if os.path.exists(t):
        open(os.path.join(OUT, f"{r}_gpu_tests.txt"), "w").write(open(t).read())
    launches(r)
    leaf_ncu(r)
    merge_ncu(r)


if __name__ == "__main__":
    main()
