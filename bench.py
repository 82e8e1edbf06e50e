"""Benchmark: sampled-nnz SGD updates/sec of the SGD_Tucker training epoch.

Metric (BASELINE.json / BASELINE.md section 2): one unit is one (nonzero, mode)
gradient visit; units per epoch = N * (M + nnz_train); throughput =
units / (core_s + factor_s), RMSE evaluation excluded (trainer.cpp:94-107).
A "step" is one training epoch (core phase + factor phase) over the resident
training tensor.

Workload (default): BASELINE config 3 (configs[2]), the largest configuration
that runs on one GPU -- 1,000,000 x 1,000,000 x 100,000 x 50, 500M nonzeros,
Zipf(1.05) on modes 1-3, uniform mode 4, planted J_n = R_core = 8 teacher plus
N(0, 0.05^2) noise, 90/10 split (450M training nonzeros), J = R = 8,
M = 262,144.  --config 2|4|5 selects the others.  The tensor is synthetic
(SURVEY.md 8(d) generator): the GPU arm draws it on the device
(paper_2012_03550_b200/synth.py -> sgdt_synth), the reference arm draws the
identical tensor on the host (oracle/synth_host.cpp) so that it never loads a
product library or touches the GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference runs the reference's own CPU implementation (oracle/_ref: the
unmodified reference sources compiled in place) on the SAME full training
tensor, Strategy::Improved on every host thread, through its timed_epochs loop
(eval.cpp:201-223).  One config 3 epoch takes minutes on the CPU, so the epoch
counts are capped by a wall-clock budget (--ref-budget); the line states how
many epochs were timed and how many were asked for.
"""
from __future__ import annotations

import argparse
import glob
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=3, choices=[2, 3, 4, 5])
    p.add_argument("--scale", type=float, default=1.0,
                   help="fraction of the config's nnz (debug only; 1.0 for reported runs)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=0, help="override the per-config CPU sample size")
    p.add_argument("--ref-budget", type=float, default=150.0,
                   help="wall-clock seconds of reference epochs (--impl reference)")
    p.add_argument("--row-fraction", type=float, default=1.0,
                   help="FactorHyper::row_fraction of our arm (diagnostics; the headline uses 1.0)")
    p.add_argument("--sharded", action="store_true",
                   help="use the multi-GPU (sharded) driver even on one rank")
    p.add_argument("--core", choices=["replicated", "sharded"], default="replicated",
                   help="multi-GPU core phase: Psi slices + peer-reduced partials, or replicated")
    return p.parse_args()


HYPER = dict(lr_a=0.01, lr_b=0.01, reg_a=0.01, reg_b=0.01, seed=1)
BATCH_M = {2: 65536, 3: 262144, 4: 65536, 5: 262144}
# cpu_baseline sample of our arm (nonzeros; a bounded 10-30 s leg): the
# reference's per-unit cost is prod(J) FMAs (dense core).
CPU_SAMPLE = {2: 3_000_000, 3: 4_000_000, 4: 0, 5: 100_000}
REF_UNAVAILABLE = {4: "the reference rejects config 4: Shape overflows 64 bits (1e5^4 x 1e3, sptensor.cpp:34-35) "
                      "and prod J = 16^5 exceeds kMaxCoreElems (model.hpp:25)"}
L2_NOTE = "inputs larger than L2: the COO record copies (N+1 copies x 4(N+1) B x nnz) exceed the 126 MB L2"


def init_stats(cfg, spec):
    """Model init.  The paper's N(0.5, 0.1^2) puts the initial xhat near
    R (J/2)^N = 156 at J = R = 10 against ratings 1..5, and lr 0.01 SGD
    diverges for some draws of it; config 2 uses N(0.3, 0.1^2) (xhat ~ 27,
    converges for every seed tried).  Configs 3-5 use N(0, sigma^2) at the
    teacher's unit-variance scale."""
    if cfg == 2:
        return 0.3, 0.1
    return 0.0, spec.unit_sigma


def config_spec(cfg, scale):
    from paper_2012_03550_b200 import synth  # pure Python (no library load)
    spec = synth.CONFIGS[cfg]
    if scale != 1.0:
        spec = synth.scaled(spec, scale ** (1.0 / len(spec.dims)), int(spec.nnz * scale))
    return spec


def units_per_epoch(order, m, nnz):
    return order * (m + nnz)


def bytes_per_unit(order, R):
    """B_u = 4(N+1) + 4(N-1)R: one u32/fp32 COO record + N-1 gathered rows of R fp32."""
    return 4 * (order + 1) + 4 * (order - 1) * R


def n_train(nnz, test_fraction=0.1):
    return nnz - int(round(test_fraction * nnz))


def workload(cfg, spec, m, row_fraction):
    """The `config` object of the JSON line -- identical in both arms."""
    order = len(spec.dims)
    J = R = spec.teacher_j
    nt = n_train(spec.nnz, spec.test_fraction)
    mean, sd = init_stats(cfg, spec)
    units = units_per_epoch(order, m, nt) if row_fraction == 1.0 else int(order * (m + row_fraction * nt))
    return {"workload": f"config{cfg}", "dims": list(spec.dims), "zipf": list(spec.zipf),
            "values": "ratings 1-5" if spec.values == "ratings" else f"teacher + N(0, {spec.noise}^2)",
            "nnz_total": spec.nnz, "nnz_train": nt, "split": "90/10 train_test_split, Rng(seed + 7)",
            "J": J, "R": R, "batch_m": m, "row_fraction": row_fraction, "units_per_step": units,
            "lr": HYPER["lr_a"], "reg": HYPER["reg_a"], "init": f"N({mean:.4g}, {sd:.4g}^2)", "seed": HYPER["seed"],
            "l2": L2_NOTE}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def build_id():
    """Hash of the CUDA sources and the C-ABI header: stamps the ncu traffic
    file so the bench only reports traffic measured on this build."""
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2012_03550_b200", "csrc", "*.cu*"))) + \
        [os.path.join(ROOT, "include", "sgdt.h")]
    for f in files:
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def factor_build_id():
    """Hash of the sources that shape the factor kernels' memory traffic (the
    kernels, the shared device helpers and the record layout / chunk schedule in
    the session): stamps profiles/factor_traffic.json, so a change to another
    phase (core, sampler, eval) does not make the factor capture stale."""
    h = hashlib.sha256()
    for name in ("sgdt_factor.cu", "sgdt_internal.cuh", "sgdt_session.cu"):
        h.update(name.encode())
        h.update(open(os.path.join(ROOT, "paper_2012_03550_b200", "csrc", name), "rb").read())
    return h.hexdigest()[:16]


def cpu_info():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return model, cores


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        os.unlink(self.path)
        rows = [[x.strip() for x in r] for r in rows if len(r) >= 7]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def make_data(cfg: int, scale: float, device):
    from paper_2012_03550_b200 import synth
    spec = config_spec(cfg, scale)
    t0 = time.time()
    train, test, _ = synth.generate(spec, device)
    return dict(spec=spec, train=train, test=test, gen_s=time.time() - t0)


def init_model(dims, J, R, mean, sd, seed):
    rs = np.random.default_rng(seed)
    B = [rs.normal(mean, sd, (J, R)) for _ in dims]
    A = [rs.normal(mean, sd, (d, J)) for d in dims]
    return A, B


def cpu_sample_run(cfg, spec, trc, trv, m, sample, threads):
    """Our arm's cpu_baseline: the reference (oracle/_ref) on a bounded uniform
    subsample of the training tensor, 1 timed epoch after 1 warm-up."""
    from oracle import oracle_py as O
    import ctypes as C
    rs = np.random.default_rng(12345)
    S = min(len(trv), sample)
    pick = np.sort(rs.choice(len(trv), S, replace=False))
    order = len(spec.dims)
    J = R = spec.teacher_j
    mm = min(m, S)
    Jv = np.array([J] * order, np.uint32)
    model, cores = cpu_info()
    desc = (f"{S:,} of {len(trv):,} training nonzeros of config {cfg} (uniform random subset, same shape), "
            f"M={mm}, 1 timed epoch after 1 warm-up, Strategy::Improved, {threads} threads, {model}")
    if not O.ref_available():
        raise RuntimeError("oracle/_ref is not built")
    t = O.RefTensor(spec.dims, trc[pick], trv[pick])
    sec = C.c_double()
    mean, sd = init_stats(cfg, spec)
    rc = O.ref().ref_time_epochs(t.h, Jv, R, HYPER["lr_a"], HYPER["lr_b"], HYPER["reg_a"], mm, 2, threads,
                                 1, 1, HYPER["seed"], mean, sd, C.byref(sec))
    if rc != 0:
        raise RuntimeError(f"reference epoch failed: {rc}")
    return {"value": units_per_epoch(order, mm, S) / sec.value, "unit": "updates/s", "cores": threads,
            "kind": "reference", "sample": desc, "cpu_model": model}


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation on the same full tensor.  Loads
    only oracle/ libraries (host generator, host split, the compiled
    reference); never imports torch or touches the GPU."""
    if rank != 0:
        return 0
    cfg = args.config
    if cfg in REF_UNAVAILABLE:
        print(json.dumps({"impl": "reference", "unavailable": REF_UNAVAILABLE[cfg]}), flush=True)
        return 0
    import ctypes as C
    from oracle import oracle_py as O
    from oracle import synth_oracle as S
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the compiled reference) is not built"}),
              flush=True)
        return 0
    spec = config_spec(cfg, args.scale)
    order = len(spec.dims)
    J = R = spec.teacher_j
    m = BATCH_M[cfg]
    model_name, threads = cpu_info()
    t0 = time.time()
    coords, values = S.synth_host(spec.dims, spec.zipf, spec.nnz, spec.teacher_j, spec.teacher_r,
                                  spec.values == "ratings", spec.noise, spec.seed, threads)
    t1 = time.time()
    _, tr = S.split_ids_host(spec.nnz, spec.test_fraction, spec.seed + 7)
    trc, trv = coords[tr], values[tr]
    del coords, values, tr
    t2 = time.time()
    t = O.RefTensor(spec.dims, trc, trv)  # the reference CooTensor constructor
    del trc, trv
    t3 = time.time()
    Jv = np.array([J] * order, np.uint32)
    secs = np.zeros(max(args.steps, 1))
    nw, nt = C.c_size_t(), C.c_size_t()
    mean, sd = init_stats(cfg, spec)
    rc = O.ref().ref_time_epochs_budget(t.h, Jv, R, HYPER["lr_a"], HYPER["lr_b"], HYPER["reg_a"], m, 2, threads,
                                        args.warmup, max(args.steps, 1), HYPER["seed"], mean, sd, args.ref_budget,
                                        secs, C.byref(nw), C.byref(nt))
    if rc != 0:
        print(json.dumps({"impl": "reference", "unavailable": f"reference epochs failed with code {rc}"}), flush=True)
        return 0
    timed = secs[:nt.value]
    med = float(np.median(timed))
    cfgd = workload(cfg, spec, m, 1.0)
    value = cfgd["units_per_step"] / med
    sample = (f"the full config {cfg} training tensor ({cfgd['nnz_train']:,} nonzeros, generated on the host by "
              f"oracle/synth_host.cpp, identical to the device generator's); timed_epochs loop (eval.cpp:201-223), "
              f"Strategy::Improved, {threads} threads on {model_name}; median of {nt.value} timed epoch(s) after "
              f"{nw.value} warm-up (asked: {args.steps} after {args.warmup}; capped by a {args.ref_budget:.0f} s "
              f"budget, one epoch takes {timed[0]:.1f} s)")
    line = {
        "metric": "sampled-nnz SGD updates/sec", "value": value, "unit": "updates/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": int(nt.value), "warmup": int(nw.value), "steps_requested": args.steps,
        "warmup_requested": args.warmup, "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Zipf/uniform indices, planted teacher; no dataset)",
        "gpu_launches": 0, "config": cfgd,
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": model_name},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "run": {"epoch_s": [float(x) for x in timed], "data_gen_s": t1 - t0, "split_s": t2 - t1,
                "tensor_build_s": t3 - t2},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpp_dropin_e2e(cfg, spec, trc, trv, m, warmup, steps):
    """End to end through the C++ drop-in (libsptucker_b200.so): a
    sptucker::CooTensor built from the host arrays, then the reference's
    timed_epochs loop (eval.cpp:201-223) -- update_core_epoch +
    update_factor_epoch on a host fp64 TuckerModel, host wall clock per epoch,
    median -- through paper_2012_03550_b200/cpp/tools/bench_shim.cpp."""
    import ctypes as C
    so = os.path.join(ROOT, "paper_2012_03550_b200", "lib", "libsptucker_bench.so")
    L = C.CDLL(so)
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    L.sptb_timed_epochs.argtypes = [C.c_int, u32p, C.c_uint64, u32p, f64p, u32p, C.c_uint32, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                    C.c_double, f64p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    order = len(spec.dims)
    J = R = spec.teacher_j
    mean, sd = init_stats(cfg, spec)
    secs = np.zeros(max(steps, 1))
    h2d, d2h, build = C.c_uint64(), C.c_uint64(), C.c_double()
    err = C.create_string_buffer(512)
    rc = L.sptb_timed_epochs(order, np.ascontiguousarray(spec.dims, np.uint32), len(trv),
                             np.ascontiguousarray(trc, np.uint32).reshape(-1), np.ascontiguousarray(trv),
                             np.full(order, J, np.uint32), R, HYPER["lr_a"], HYPER["lr_b"], HYPER["reg_a"], m,
                             warmup, max(steps, 1), HYPER["seed"], mean, sd, secs, C.byref(h2d), C.byref(d2h),
                             C.byref(build), err, 512)
    if rc != 0:
        raise RuntimeError(err.value.decode(errors="replace"))
    units = units_per_epoch(order, m, len(trv))
    med = float(np.median(secs))
    n = max(steps, 1)
    return {"value": units / med, "unit": "updates/s", "ms_per_step": med * 1e3,
            "h2d_bytes_per_step": int(h2d.value) // n, "d2h_bytes_per_step": int(d2h.value) // n,
            "path": "C++ drop-in (libsptucker_b200.so): sptucker::CooTensor + the reference's timed_epochs loop "
                    "(update_core_epoch + update_factor_epoch on a host fp64 TuckerModel per epoch; model and sample "
                    "pool stay device-resident between calls, B / A / pool deltas copied back every epoch), "
                    "host wall clock, median",
            "epoch_ms": [float(x) * 1e3 for x in secs], "tensor_build_s": build.value}


def factor_traffic(cfg, mode_ms, peak):
    """ncu DRAM / L2 bytes per factor-mode launch group of THIS build
    (profiles/factor_traffic.json, written by scripts/ncu_factor_traffic.py,
    stamped with factor_build_id()).  None when the file is for another build."""
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "factor_traffic.json")))
    except Exception:
        return None
    if tj.get("build") != factor_build_id():
        return {"stale": f"profiles/factor_traffic.json is for factor build {tj.get('build')}, this is {factor_build_id()}"}
    c = tj.get(f"config{cfg}")
    if not c:
        return None
    dram = c["dram_bytes_per_mode"]
    avg_ms = sum(mode_ms) / len(mode_ms)
    return {"dram_bytes": dram, "l2_bytes": c.get("l2_bytes_per_mode"),
            "dram_gbs": dram / (avg_ms * 1e-3) / 1e9, "dram_frac": dram / (avg_ms * 1e-3) / 1e9 / peak,
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum (build {tj['build']})"}


def run_sharded(args, rank, world, local_rank):
    """N GPUs: factor phase sharded over ranks (partition_even slices of every
    mode order, peer-published rows, rank-ordered boundary merge), core phase
    sharded (partition_even Psi slices, rank-ordered peer-reduced column
    partials) or replicated -- paper_2012_03550_b200/distributed.py.  Total
    work is the config's epoch, so scaling is strong."""
    import torch
    import torch.distributed as dist
    from paper_2012_03550_b200 import distributed as D
    from paper_2012_03550_b200 import sgdt
    torch.cuda.set_device(local_rank)
    if "RANK" not in os.environ:  # --sharded without torchrun: a world of one
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    group = D.TorchGroup()
    cfg = args.config
    data = make_data(cfg, args.scale, torch.device("cuda", local_rank))
    spec = data["spec"]
    order = len(spec.dims)
    J = R = spec.teacher_j
    m = BATCH_M[cfg]
    trc, trv = data["train"]
    nnz = len(trv)
    t0 = time.time()
    s = D.ShardedSession(spec.dims, trc, trv, [J] * order, R, rank, world, test=data["test"],
                         device=local_rank)
    setup_s = time.time() - t0
    A, B = init_model(spec.dims, J, R, *init_stats(cfg, spec), HYPER["seed"])
    s.set_model(A, B)
    s.seed(HYPER["seed"] + 1)
    ch = sgdt.CoreHyper(HYPER["lr_b"], HYPER["reg_b"], m, 0, 0)
    fh = sgdt.FactorHyper(HYPER["lr_a"], HYPER["reg_a"], 1.0)
    D.connect_peers(s, group)
    dist.barrier()
    D.run_epochs_p2p(s, group, ch, fh, args.warmup, core=args.core)
    stream = torch.cuda.ExternalStream(s.stream)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = s.launch_count()
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        D.run_epochs_p2p(s, group, ch, fh, args.steps, core=args.core)
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    launches = s.launch_count() - launches0
    t = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    units = units_per_epoch(order, m, nnz)
    value = units * args.steps / (elapsed_ms * 1e-3)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hA, hB = [pin(a) for a in A], [pin(b) for b in B]
        oA = [torch.empty(a.shape, dtype=torch.float64).pin_memory().numpy() for a in A]
        oB = [torch.empty(b.shape, dtype=torch.float64).pin_memory().numpy() for b in B]
        s.get_model((hA, hB))
        h2d = sum(a.nbytes for a in hA) + sum(b.nbytes for b in hB)
        d2h = sum(a.nbytes for a in oA) + sum(b.nbytes for b in oB)
        for _ in range(args.warmup):  # untimed
            s.set_model(hA, hB)
            D.run_epochs_p2p(s, group, ch, fh, 1, core=args.core)
            s.get_model((oA, oB))
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            s.set_model(hA, hB)
            D.run_epochs_p2p(s, group, ch, fh, 1, core=args.core)
            s.get_model((oA, oB))
            hA, oA = oA, hA
            hB, oB = oB, hB
        ev1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item()) / args.steps
        e2e = {"value": units / (e_ms * 1e-3), "unit": "updates/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "per rank: sgdt_set_model (fp64 pinned host) + sharded epoch + sgdt_get_model (fp64 pinned host)"}
    rmse = s.eval(1)[0]
    if rank == 0:
        cfgd = workload(cfg, spec, m, 1.0)
        line = {
            "metric": "sampled-nnz SGD updates/sec", "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Zipf/uniform indices, planted teacher; no dataset)",
            "config": cfgd,
            "run": {"parallelism": f"{world} GPUs: factor phase sharded (partition_even slices of every mode "
                                   "order; finalised rows stored into every peer's A/Q over NVLink P2P; rank-ordered "
                                   f"boundary merge); core phase {args.core}",
                    "test_rmse_after": rmse, "setup_s": setup_s, "data_gen_s": data["gen_s"]},
            "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2012_03550_b200 import sgdt
    if world > 1 or args.sharded:
        return run_sharded(args, rank, world, local_rank)
    torch.cuda.set_device(local_rank)
    cfg = args.config
    data = make_data(cfg, args.scale, torch.device("cuda", local_rank))
    spec = data["spec"]
    order = len(spec.dims)
    J = R = spec.teacher_j
    m = BATCH_M[cfg]
    trc, trv = data["train"]
    nnz = len(trv)

    t0 = time.time()
    s = sgdt.Session(spec.dims, trc, trv, [J] * order, R, test=data["test"], device=local_rank)
    setup_s = time.time() - t0
    A, B = init_model(spec.dims, J, R, *init_stats(cfg, spec), HYPER["seed"])
    s.set_model(A, B)
    s.seed(HYPER["seed"] + 1)
    ch = sgdt.CoreHyper(HYPER["lr_b"], HYPER["reg_b"], m, 0, 0)
    fh = sgdt.FactorHyper(HYPER["lr_a"], HYPER["reg_a"], args.row_fraction)
    for _ in range(args.warmup):
        s.run_epochs(ch, fh, 1)

    stream = torch.cuda.ExternalStream(s.stream)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = s.launch_count()
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        s.run_epochs(ch, fh, args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = s.launch_count() - launches0
    elapsed_ms = ev0.elapsed_time(ev1)
    timing = s.last_timing()  # per-phase means over the K timed epochs (CUDA events, session stream)
    cfgd = workload(cfg, spec, m, args.row_fraction)
    units = cfgd["units_per_step"]
    value = units * args.steps / (elapsed_ms * 1e-3)
    ms_per_step = elapsed_ms / args.steps

    # roofline of the dominant kernel: the factor phase's launches of one mode
    bu = bytes_per_unit(order, R)
    mode_ms = [timing.factor_mode_ms[n] for n in range(order)]
    avg_mode_ms = sum(mode_ms) / order
    achieved_gbs = nnz * bu / (avg_mode_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    traffic = factor_traffic(cfg, mode_ms, peak)
    # bytes outside B_u, per epoch: the mode-n row traffic of the
    # factor phase (read a and Q^(n), write a and Q^(n) per non-empty row) and
    # the Q^(k) refresh at the end of the core phase
    rows_nonempty = [int(np.count_nonzero(np.bincount(trc[:, n], minlength=spec.dims[n] + 1)))
                     for n in range(order)]
    overhead = {"mode_rows": sum(4 * (2 * J + 2 * R) * r for r in rows_nonempty),
                "q_refresh": sum(4 * d * (J + R) for d in spec.dims),
                "b_u_total": units * bu}

    rmse = s.eval(1)[0]

    # end to end through the C-ABI with host buffers: H2D model, epoch, D2H model
    e2e = e2e_cabi = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        hA, hB = [pin(a) for a in A], [pin(b) for b in B]
        oA = [torch.empty(a.shape, dtype=torch.float64).pin_memory().numpy() for a in A]
        oB = [torch.empty(b.shape, dtype=torch.float64).pin_memory().numpy() for b in B]
        s.get_model((hA, hB))  # continue from the trained state
        h2d = sum(a.nbytes for a in hA) + sum(b.nbytes for b in hB)
        d2h = sum(a.nbytes for a in oA) + sum(b.nbytes for b in oB)
        for _ in range(args.warmup):  # untimed: first-call staging allocation, page-ins
            s.run_epochs_host(ch, fh, 1, (hA, hB), (oA, oB))
            hA, oA = oA, hA
            hB, oB = oB, hB
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            s.run_epochs_host(ch, fh, 1, (hA, hB), (oA, oB))
            hA, oA = oA, hA
            hB, oB = oB, hB
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.steps
        e2e_cabi = {"value": units / (e_ms * 1e-3), "unit": "updates/s", "ms_per_step": e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "sgdt_run_epochs_host(1): fp64 pinned host model in -> epoch -> fp64 pinned host model out"}
    s.close()  # the device memory goes to the drop-in's own session
    if not args.no_e2e:
        try:
            e2e = cpp_dropin_e2e(cfg, spec, trc, trv, m, args.warmup, args.steps)
        except Exception as exc:  # reported; the C-ABI figure stands in
            e2e = dict(e2e_cabi or {}, error=f"C++ drop-in leg failed: {type(exc).__name__}: {exc}")

    cpu = None
    if rank == 0 and cfg in REF_UNAVAILABLE and not args.no_cpu_baseline:
        cpu = {"value": None, "unit": "updates/s", "cores": 0, "kind": "unavailable", "sample": REF_UNAVAILABLE[cfg]}
    elif rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample_run(cfg, spec, trc, trv, m, args.cpu_sample or CPU_SAMPLE[cfg], cpu_info()[1])
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": "updates/s", "cores": 0, "kind": "unavailable",
                   "sample": f"{type(exc).__name__}: {exc}"}

    roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s", "frac": achieved_gbs / peak,
            "traffic": traffic.get("dram_bytes") if traffic else None,
            "frac_basis": "algorithmic: B_u x nnz per factor-mode launch group / its mean CUDA-event time; the "
                          "gathered Q rows are served from L1/L2, so this can exceed 1 -- dram_frac is the HBM share",
            "kernel": ("factor_staged_kernel / factor_chunk_kernel" if (R + 3) // 4 * 4 <= 12
                       else "factor_group_kernel") + " + factor_split_kernel (one mode)",
            "bytes_per_unit": bu, "units_per_launch": nnz, "launch_ms": avg_mode_ms,
            "timed_epochs": int(timing.epochs), "peak_source": peak_src, "overhead_bytes_per_epoch": overhead}
    if traffic:
        roof.update({k: traffic[k] for k in ("dram_gbs", "dram_frac", "l2_bytes", "source") if k in traffic})
        if "stale" in traffic:
            roof["traffic_note"] = traffic["stale"]
    line = {
        "metric": "sampled-nnz SGD updates/sec", "value": value, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Zipf/uniform indices, planted teacher; no dataset)",
        "config": cfgd,
        "run": {"parallelism": "single GPU", "test_rmse_after": rmse, "data_gen_s": data["gen_s"],
                "setup_s": setup_s, "build": build_id()},
        "phase_ms": {"core": timing.core_ms, "factor": timing.factor_ms, "factor_modes": mode_ms},
        "roofline": roof,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "e2e_cabi": e2e_cabi,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
