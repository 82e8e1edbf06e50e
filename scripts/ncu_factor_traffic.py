"""Per-launch DRAM / L2 traffic of the factor kernels, for bench.py's roofline.

Run on the GPU box (one GPU, never under torchrun):
    python scripts/ncu_factor_traffic.py [configs...]      (default: 2 3 4 5)
For each BASELINE config it profiles one epoch of `bench.py --config C` with
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,
          l1tex__data_pipe_lsu_wavefronts.sum,gpu__time_duration.sum
        --cache-control none --clock-control none -k regex:factor_(chunk|staged|group)_kernel
(warm L2 between launches, as inside the timed epochs), averages the N mode
launches of the second epoch and writes profiles/factor_traffic.json stamped
with bench.factor_build_id(), so the bench reports only traffic measured on the
build it runs.  Raw CSVs go to gpurun_out/ncu_traffic_c<C>.csv.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "l1tex__data_pipe_lsu_wavefronts.sum", "gpu__time_duration.sum"]
ORDER = {2: 3, 3: 4, 4: 5, 5: 3}


def profile(cfg: int) -> dict:
    out = os.path.join(ROOT, "gpurun_out", f"ncu_traffic_c{cfg}.csv")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    n = ORDER[cfg]
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--cache-control", "none", "--clock-control", "none",
           "-k", "regex:factor_(chunk|staged|group)_kernel", "-s", str(n), "-c", str(n), "--csv",
           "--log-file", out, sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg),
           "--steps", "1", "--warmup", "1", "--no-cpu-baseline", "--no-e2e"]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=1800)
    rows = [r for r in csv.reader(open(out)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for r in rows[1:]:
        per.setdefault(r[ki], {})[r[mi]] = float(r[vi].replace(",", ""))
    launches = list(per.values())
    mean = lambda k: sum(x[k] for x in launches) / len(launches)
    return {"launches": len(launches),
            "dram_bytes_per_mode": mean("dram__bytes_read.sum") + mean("dram__bytes_write.sum"),
            "l2_bytes_per_mode": mean("lts__t_bytes.sum"),
            "l1_wavefronts_per_mode": mean("l1tex__data_pipe_lsu_wavefronts.sum"),
            "ncu_ms_per_mode": mean("gpu__time_duration.sum") / 1e6}


def main(argv):
    cfgs = [int(a) for a in argv] or [2, 3, 4, 5]
    path = os.path.join(ROOT, "profiles", "factor_traffic.json")
    try:
        tj = json.load(open(path))
    except Exception:
        tj = {}
    if tj.get("build") != bench.factor_build_id():
        tj = {}
    tj["build"] = bench.factor_build_id()
    tj["how"] = ("ncu --metrics " + ",".join(METRICS) + " --cache-control none --clock-control none, "
                 "the factor-kernel launches of the second epoch of bench.py --steps 1 --warmup 1, mean per mode")
    for c in cfgs:
        tj[f"config{c}"] = profile(c)
        print(c, tj[f"config{c}"], flush=True)
    json.dump(tj, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
