"""Benchmark: FMM evaluated points/s on B200 (BASELINE.json metric) + roofline + CPU oracle.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl fmm2d|reference]

One step = one pass of the whole hot path (rows A0-A11) over one
synthetic instance: fmm2d_build (validate, median-split tree, discs, theta-criterion
lists) + fmm2d_eval (P2M, M2M, M2L, L2L, L2P + P2P, input order) for Phi and Phi'.
Inputs (z, m) are resident in HBM before the timed region; every instance is larger
than L2 (C5: 1.6 GB of positions), so no extra L2 flush is needed.

value      = N * steps * n_gpus / max-over-ranks device time (points/s, whole job)
e2e        = the same through the C ABI with HOST buffers (pinned): H2D of z and m,
             D2H of Phi and Phi' inside the timed region
roofline   = the dominant kernel (P2P+L2P, k_near): algorithmic FP64 flops per launch
             (ordered pairs x 105 flop) / its CUDA-event time vs the
             measured FP64 peak
cpu_baseline = the oracle (oracle/, plain C++, OpenMP) on a bounded sample of the same
             workload: the C5 recipe at N = 1,562,500 (same leaf occupancy, L = 8), build +
             eval passes repeated up to about 10 s of host work

--impl reference runs the oracle itself (the reference arm for this tier) on rank 0.
Multi-GPU (torchrun, N > 1): ONE instance of the config partitioned across the ranks by
the balanced tree's level-k subtrees (strong scaling): every rank
holds the full z and m, builds its share (replicated top levels, own subtrees below,
NCCL halo exchange) and evaluates its own sources.  value = N * steps / max-over-ranks
device time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "FMM evaluated points/sec at 1/2/4/8 B200 (θ=0.5, p=17) and % FP64 roofline"
M2L_FLOPS_PER_PAIR = 1450.0       # SURVEY 8(d), p = 17
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
CENSUS = os.path.join(ROOT, "profiles", "r02", "fp64_census.json")


def census():
    try:
        return json.load(open(CENSUS))
    except Exception:
        return {}


def p2p_flops_per_pair():
    """SURVEY 8(d)'s convention: each transcendental at its libdevice FP64 instruction cost,
    measured once by ncu on a microbenchmark (tools/p2p_census.cu): 2 DFMA + DADD + DMUL per
    pair of the library-math pair body (128 at C5-like |dz|).  Falls back to the survey's
    working estimate 105 if the census is missing."""
    c = census().get("libdevice_pair", {})
    return float(c.get("flops_per_pair", 105.0)), (os.path.relpath(CENSUS, ROOT) if c else "SURVEY 8(d) working estimate")
# bounded CPU sample of a workload for the oracle: the C5 recipe at L = 8 (same leaf occupancy,
# 23.8 points per leaf), build + eval passes repeated up to about 10 s of host work
CPU_SAMPLE_N = 1_562_500
# end-to-end line: problems in flight on as many streams (FMM2D_ASYNC_HOST); the oldest is
# synchronised (its result copies complete) when a new one is issued beyond this count
E2E_IN_FLIGHT = int(os.environ.get("FMM2D_E2E_IN_FLIGHT", "3"))
CPU_SAMPLE_SECONDS = 10.0


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def hbm_peak():
    """(GB/s, source): the measured copy bandwidth of MEASURED_PEAKS.json, else the
    profiling recipe's fallback figure."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "MEASURED_PEAKS.json:hbm_gbs"
    except Exception:
        return 6544.0, "B200_PROFILING.md fallback"


def build_algorithmic_bytes(n, L, weak, strong, nboxes):
    """Algorithmic DRAM bytes of one fmm2d_build (rows A0-A3) -- what each build kernel must
    read and write at least, by the data layout of DESIGN 6.1 (records of 8 B, radix sorts
    of a 4-byte key + 8-byte payload in four 8-bit passes):
      canonicalise z (16 B in, 16 B out); x / y keys + payloads (16 + 12, 8 + 12 B);
      two stable radix sorts: 4 onesweep passes x (12 B in + 12 B out) + a 4-byte histogram
      pass, run fix-up key scans (4 B); y-list + x-list (24 B, one 8-byte bucketing pass of
      16 B, the scatter 16 B); 2 l0 global split steps of 16 B (8 B record in + out);
      the on-chip levels (both lists in, the y-list out: 24 B); the final pass (y-list 8,
      y-rank -> idx 8, coordinates 16 in; perm 4 + source row 32 out); lists: 12 B per
      CSR entry (slot written + read, CSR written) + 24 B per box (disc)."""
    l0 = L
    for l in range(max(0, L - 4), L):
        if -(-n // 4 ** l) <= 2048:
            l0 = l
            break
    per_pt = {"canon": 32, "keys": 28 + 20, "radix_sorts": 2 * (4 * 24 + 4), "fix_runs": 8,
              "lists_xy": 24 + 16 + 16, "split_steps": 2 * l0 * 16, "local_levels": 24 if l0 < L else 0,
              "finish": 68}
    comp = {k: float(v) * n for k, v in per_pt.items()}
    comp["connectivity"] = 12.0 * (weak + strong) + 24.0 * nboxes
    return comp, l0


def fp64_peak():
    """(TFLOP/s, source).  MEASURED_PEAKS.json if it has an FP64 entry; else, for a path bound
    by plain FP64 ALU work, the peak derived from the unit counts and clock (B200_PROFILING.md:
    148 SMs, 64 FP64 lanes each, 1.965 GHz clocks.max.sm) = 37.2 TFLOP/s.  The measured DFMA
    loop and cuBLAS DGEMM figures are reported beside it (roofline.peaks)."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("fp64_tflops", "fp64_tflops_sustained"):
            if k in mp:
                return float(mp[k]), "MEASURED_PEAKS.json:" + k
    except Exception:
        pass
    return NOMINAL_FP64_TFLOPS, "derived: 148 SM x 64 FP64 lanes x 2 flop x 1.965 GHz (unit counts and clock)"


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region, in-process through NVML
    (pynvml; spawning nvidia-smi every 200 ms stalled the CUDA driver and inflated the
    timed steps).  Falls back to nvidia-smi only if NVML cannot be loaded."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap")]

    def __init__(self, device: int, period: float = 0.1):
        self.device = device
        self.period = period
        self.samples = []           # (sm_mhz, max_mhz, [reasons])
        self.source = None
        self._stop = threading.Event()
        self._t = None

    def _nvml_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.device < len(ids) and ids[self.device].isdigit():
                return int(ids[self.device])
        return self.device

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self._nvml_index())
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            masks = [(name, getattr(N, attr)) for name, attr in self.REASONS]

            def sample():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                return (float(sm), float(mx), [name for name, m in masks if r & m])
            self.source = "nvml"
        except Exception:
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")

            def sample():
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                v = [s.strip() for s in out]
                return (float(v[0]), float(v[1]),
                        [self.REASONS[i][0] for i in range(4) if v[2 + i].lower() == "active"])
            self.source = "nvidia-smi"

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(sample())
                except Exception:
                    pass
                self._stop.wait(self.period)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({r for s in self.samples for r in s[2]}), "samples": len(self.samples),
                "source": self.source}


def k_near_traffic(cfg, default_cfg):
    """DRAM bytes per k_near launch from the committed ncu --set full capture
    (profiles/traffic.json) -- only for the configuration it was captured on."""
    if not default_cfg:
        return None, None
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["k_near"]
        return float(d["dram_bytes_per_launch"]), d["source"]
    except Exception:
        return None, None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


ONE_THREAD_N = 390_625          # C5 recipe at L = 7: the same leaf occupancy (23.8), one pass


def oracle_one_thread(cfg):
    """The oracle on ONE host thread (OMP_NUM_THREADS=1, a child process): one build + eval
    of the C5 recipe at N = 390,625 (same leaf occupancy), points/s."""
    code = ("import sys, time; sys.path.insert(0, %r); import oracle, workloads as W; "
            "z, m = W.make(%r, %d, %r, seed=W.SEED_BASE + 78); L = oracle.nlevels(%d, %d); "
            "t = time.perf_counter(); P = oracle.plan(z, %r, L); P.eval(m, %d); "
            "print(time.perf_counter() - t)") % (ROOT, cfg.dist, ONE_THREAD_N, cfg.strengths, ONE_THREAD_N,
                                                  cfg.leaf_target, cfg.theta, cfg.p)
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, OMP_NUM_THREADS="1"))
        dt = float(r.stdout.strip().splitlines()[-1])
    except Exception as e:                       # report, never fail the bench line over it
        return {"error": str(e)[:200]}
    return {"value": ONE_THREAD_N / dt, "unit": "points/s", "cores": 1, "seconds": dt,
            "sample": f"{cfg.dist} N={ONE_THREAD_N} (same leaf occupancy as {cfg.name}), one build+eval"}


def parity_record(default_cfg):
    """The committed whole-problem parity log of the bench's own configuration (C5)."""
    if not default_cfg:
        return None
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02", "full_parity_C5.json")))
    except Exception:
        return None
    return {"source": "profiles/r02/full_parity_C5.json (tools/full_parity.py; tests/test_gpu_fullsize.py)",
            "levels_bit_exact": len(d["levels_compared"]), "list_entries_bit_exact": d["entries_compared"],
            "phi_normwise": d["phi"]["norm"], "phi_pointwise": d["phi"]["point"],
            "dphi_normwise": d["dphi"]["norm"], "dphi_pointwise": d["dphi"]["point"],
            "pointwise_floor": f"{d['pt_floor']:g} max|ref|", "bar": 1e-12}


def cpu_baseline(cfg, seconds_hint=True):
    """Oracle (plain C++ + OpenMP) on a bounded sample of the same workload."""
    import oracle
    n = min(cfg.n, CPU_SAMPLE_N)
    z, m = W.make(cfg.dist, n, cfg.strengths, seed=W.SEED_BASE + 77)
    L = oracle.nlevels(n, cfg.leaf_target)
    # build + eval passes until about CPU_SAMPLE_SECONDS of work (at least one, at most 8)
    passes, dt = 0, 0.0
    while passes < 1 or (dt < CPU_SAMPLE_SECONDS and passes < 8):
        t0 = time.perf_counter()
        P = oracle.plan(z, cfg.theta, L)
        P.eval(m, cfg.p)
        dt += time.perf_counter() - t0
        passes += 1
    cores = _env_int("OMP_NUM_THREADS", os.cpu_count() or 1)
    return {"value": n * passes / dt, "unit": "points/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{cfg.dist} N={n} (L={L}, same leaf occupancy as {cfg.name}), theta={cfg.theta}, "
                      f"p={cfg.p}: {passes} build+eval passes, {dt:.1f} s",
            "one_thread": oracle_one_thread(cfg)}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    n = min(cfg.n, CPU_SAMPLE_N)
    z, m = W.make(cfg.dist, n, cfg.strengths, seed=W.SEED_BASE + 77)
    L = oracle.nlevels(n, cfg.leaf_target)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        P = oracle.plan(z, cfg.theta, L)
        P.eval(m, cfg.p)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    T = float(np.sum(times))
    value = n * len(times) / T
    cores = _env_int("OMP_NUM_THREADS", os.cpu_count() or 1)
    line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{cfg.name} recipe at N={n} (bounded CPU sample)", "n": n, "theta": cfg.theta,
                       "p": cfg.p, "leaf_target": cfg.leaf_target, "levels": L + 1},
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle",
                             "sample": f"{cfg.dist} N={n}, one oracle build+eval per step"},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on this node and return its exit code; rank 0 prints the line.
    Fails loudly if the node has fewer than N GPUs."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} needs {n} CUDA devices, this node has {have}", file=sys.stderr, flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=None, help="override N (same recipe)")
    ap.add_argument("--impl", default="fmm2d", choices=["fmm2d", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-optional", action="store_true", help="skip the optional-steps lines")
    ap.add_argument("--rr-exchange", action="store_true", help="FMM2D_RR_EXCHANGE (P:370-377; one GPU)")
    ap.add_argument("--parent-merge", action="store_true", help="FMM2D_PARENT_MERGE (P:364-370)")
    ap.add_argument("--symmetric-p2p", action="store_true", help="FMM2D_SYMMETRIC_P2P (one GPU)")
    ap.add_argument("--overlap", action="store_true", help="FMM2D_OVERLAP: expansions concurrent with P2P (one GPU)")
    args = ap.parse_args()
    cfg = W.CONFIGS[args.config]
    if args.n:
        cfg = W.Config(cfg.name, args.n, cfg.dist, cfg.strengths, cfg.theta, cfg.p, cfg.leaf_target)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world if "WORLD_SIZE" in os.environ else args.gpus)
        return

    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")

    import torch
    import torch.distributed as dist
    from paper_1006_2269_b200 import Fmm2d
    from paper_1006_2269_b200.dist import shared_nccl_id

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
        # one line per rank on stderr (the JSON line stays rank 0's only stdout line)
        print(f"bench.py: rank {rank} of {world} on cuda:{local_rank} ({torch.cuda.get_device_name(dev)}), "
              f"NCCL process group up", file=sys.stderr, flush=True)

    def barrier():
        if world > 1:
            dist.barrier()

    # inputs resident in HBM (one instance; every rank holds all of it)
    z_np, m_np = W.make(cfg.dist, cfg.n, cfg.strengths, seed=W.SEED_BASE + 4)
    nccl_id = shared_nccl_id() if world > 1 else None
    shard_kw = dict(nranks=world, rank=rank, nccl_id=nccl_id) if world > 1 else {}
    if args.rr_exchange:
        shard_kw["rr_exchange"] = True
    if args.parent_merge:
        shard_kw["parent_merge"] = True
    if args.symmetric_p2p:
        shard_kw["symmetric_p2p"] = True
    if args.overlap:
        shard_kw["overlap"] = True
    z = torch.from_numpy(z_np).to(dev)
    m = torch.from_numpy(m_np).to(dev)
    real = cfg.strengths == "real"
    phi = torch.empty(cfg.n, dtype=torch.complex128, device=dev)
    dphi = torch.empty(cfg.n, dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan = Fmm2d(z, theta=cfg.theta, p=cfg.p, leaf_target=cfg.leaf_target, real_strengths=real,
                     stream=stream, **shard_kw)
        plan.eval(m, phi, dphi)
        return plan

    # warm-up
    last = None
    for _ in range(args.warmup):
        if last is not None:
            last.close()
        last = step()
    torch.cuda.synchronize()
    info = last.stats() if last is not None else {}
    if last is not None:
        last.close()
    L = int(info.get("L", 0))

    # timed region
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    plan = None
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            if plan is not None:
                plan.close()          # each step: free the previous plan, build + evaluate anew
            plan = step()
        e1.record(stream)
        torch.cuda.synchronize()
    host_ms = (time.perf_counter() - h0) * 1e3
    barrier()
    ms = e0.elapsed_time(e1)
    st = plan.stats()
    L = int(st.get("L", L))
    plan.close()
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = cfg.n * args.steps / (ms_max / 1e3)          # one instance of N points per step

    # per-phase breakdown + roofline of the dominant kernel (k_near) on one extra pass
    phase = phase_times(z, m, phi, dphi, cfg, real, stream, shard_kw)
    peak, peak_src = fp64_peak()
    pairs = st.get("p2p_pairs", 0.0)
    near_ms = phase["near_ms"]
    fpp, fpp_src = p2p_flops_per_pair()
    achieved = pairs * fpp / (near_ms / 1e3) / 1e12
    traffic, traffic_src = k_near_traffic(cfg, args.config == "C5" and not args.n and world == 1
                                          and not args.rr_exchange and not args.parent_merge
                                          and not args.symmetric_p2p)
    nleaf = 4 ** L if L else 1
    algo_bytes = 32.0 * cfg.n * 2 + 4.0 * cfg.n + 288.0 * nleaf        # rows in, Phi/Phi' out, perm, locals
    cen = census()
    roof = {"bound": "alu", "kernel": "k_near (P2P+L2P)", "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": algo_bytes,
            "flops_per_launch": pairs * fpp, "pairs_per_launch": pairs,
            "peak_source": peak_src,
            "flop_convention": f"{fpp:g} FP64 flop per ordered P2P pair: the libdevice pair body's executed "
                               f"2 DFMA + DADD + DMUL, ncu census ({fpp_src}; SURVEY 8(d))",
            "peaks": cen.get("peaks_tflops")}
    kn = cen.get("k_near")
    if kn and "flops_per_pair" in kn:
        ex = pairs * kn["flops_per_pair"] / (near_ms / 1e3) / 1e12
        roof["executed"] = {"flops_per_pair": kn["flops_per_pair"], "tflops": ex, "frac_of_peak": ex / peak,
                            "fp64_pipe_pct": kn.get("fp64_pipe_pct"), "source": os.path.relpath(CENSUS, ROOT),
                            "note": "the kernel's own executed FP64 flops (table-driven log/Arg/rcp need fewer "
                                    "than libdevice's); the FP64-pipe utilisation is clock-independent"}
    if roof["frac"] > 1.0:
        roof["frac_note"] = ("above 1 under the survey's convention: the kernel's table-driven pair body does the "
                             "libdevice-equivalent work of a pair in fewer executed FP64 operations; see 'executed' "
                             "(the kernel's own flops against the same peak) and 'pipe_limits'")
    try:       # what the FP64 pipe delivers per operand form (tools/fp64_mix.cu, measured on this pool's B200)
        mix = json.load(open(os.path.join(ROOT, "profiles", "r02", "fp64_mix.json")))["fp64_rate_fraction_of_nominal"]
        roof["pipe_limits"] = {"dfma_shared_operands": mix["dfma_shared_operands"],
                               "dfma_three_distinct_registers": mix["dfma_distinct_operands"],
                               "source": "profiles/r02/fp64_mix.json (fraction of the nominal FP64 rate; k_near's "
                                         "operand mix sits between the two, DESIGN.md 6.4)"}
    except (OSError, KeyError, ValueError):
        pass
    weak_pairs = st.get("weak_pairs", 0.0)
    m2l_tf = weak_pairs * M2L_FLOPS_PER_PAIR / (phase["m2l_ms"] / 1e3) / 1e12 if phase["m2l_ms"] > 0 else 0.0
    # the M2L kernel against the same FP64 peak (algorithmic 1450 flop per pair, SURVEY 8(d);
    # executed flops from the ncu census)
    roof_m2l = None
    if phase["m2l_ms"] > 0 and weak_pairs > 0:
        km = cen.get("k_m2l", {})
        roof_m2l = {"bound": "alu", "kernel": "k_m2l (M2L, every level)", "unit": "TFLOP/s", "peak": peak,
                    "achieved": m2l_tf, "frac": m2l_tf / peak, "flops_per_pair": M2L_FLOPS_PER_PAIR,
                    "pairs_per_launch": weak_pairs, "flop_convention": "4p(p+1) + 12p + 40 at p = 17 (SURVEY 8(d))"}
        if "flops_per_pair" in km:
            ex = weak_pairs * km["flops_per_pair"] / (phase["m2l_ms"] / 1e3) / 1e12
            roof_m2l["executed"] = {"flops_per_pair": km["flops_per_pair"], "tflops": ex, "frac_of_peak": ex / peak,
                                    "fp64_pipe_pct": km.get("fp64_pipe_pct"), "source": os.path.relpath(CENSUS, ROOT)}
    # the build (rows A0-A3) against the HBM peak, on its algorithmic bytes
    hbm, hbm_src = hbm_peak()
    comp, l0 = build_algorithmic_bytes(cfg.n if world == 1 else cfg.n // world, L, weak_pairs,
                                       st.get("strong_leaf_pairs", 0.0), st.get("nboxes", 0.0))
    bbytes = sum(comp.values())
    build_gbs = bbytes / (phase["build_ms"] / 1e3) / 1e9 if phase["build_ms"] > 0 else 0.0
    roof_build = {"bound": "hbm", "kernels": "fmm2d_build (A0-A3: presort, split steps, on-chip levels, finish, lists)",
                  "unit": "GB/s", "achieved": build_gbs, "peak": hbm, "frac": build_gbs / hbm, "peak_source": hbm_src,
                  "algorithmic_bytes": bbytes, "components_bytes": comp, "global_split_levels": l0,
                  "traffic": None, "traffic_note": "per-kernel ncu DRAM bytes: DESIGN.md 6.1 table"}

    # the same workload with the paper's two optional steps (r/R exchange P:370-377 and parent
    # merge P:364-370, off on the headline path by reading R17): device
    # time per build + eval, same clocking rules, a short run
    optional = None
    if world == 1 and not (args.rr_exchange or args.parent_merge or args.overlap or args.symmetric_p2p) \
            and not args.no_optional:
        optional = optional_steps(z, m, phi, dphi, cfg, real, stream, steps=3, warmup=2)

    # end to end through the C ABI with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        e2e = end_to_end(z_np, m_np, cfg, real, stream, args, shard_kw)
        if world > 1:
            t = torch.tensor([e2e["ms"]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["ms"] = float(t.item())
        single = e2e.get("single_ms")
        e2e = {"value": cfg.n / (e2e["ms"] / 1e3), "unit": "points/s",
               "h2d_bytes_per_step": e2e["h2d"] * world, "d2h_bytes_per_step": e2e["d2h"] * world,
               "mode": (f"{E2E_IN_FLIGHT} problems in flight (fmm2d_build_eval, FMM2D_ASYNC_HOST, one stream each)"
                        if not shard_kw else "one problem at a time (build, then eval)")}
        if single is not None:
            e2e["single_call"] = {"value": cfg.n / (single / 1e3), "unit": "points/s", "ms": single,
                                  "mode": "one synchronous fmm2d_build_eval at a time (host buffers, latency)"}

    launches_per_step = phase["launches"]
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{cfg.name}: {cfg.dist} N={cfg.n}"
                                       + (f" partitioned over {world} GPUs" if world > 1 else " (single GPU)"),
                           "n": cfg.n, "theta": cfg.theta, "p": cfg.p, "leaf_target": cfg.leaf_target,
                           "levels": L + 1, "strengths": cfg.strengths,
                           "step": "fmm2d_build + fmm2d_eval (rows A0-A11)",
                           "l2": "inputs larger than L2 (no flush needed)",
                           "parallelism": f"subtrees{world}" if world > 1 else "single"},
                "phases_ms": phase, "host_ms_per_step": host_ms / args.steps, "eval_only_points_per_s": cfg.n / (phase["eval_ms"] / 1e3),
                "m2l_tflops": m2l_tf,
                "roofline": roof, "roofline_m2l": roof_m2l, "roofline_build": roof_build,
                "gpu_launches": launches_per_step * args.steps,
                "clocks": clk.summary(), "e2e": e2e, "optional_steps": optional,
                "stats": {"weak_pairs": weak_pairs, "p2p_pairs": pairs, "min_leaf": st.get("min_leaf"),
                          "max_leaf": st.get("max_leaf")}}
        line["parity"] = parity_record(args.config == "C5" and not args.n)
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def optional_steps(z, m, phi, dphi, cfg, real, stream, steps=3, warmup=2):
    """Points/s of build + eval with the r/R exchange and the parent merge (each alone and
    both), CUDA events on the launching stream, W untimed steps first."""
    import torch
    from paper_1006_2269_b200 import Fmm2d
    out = {"note": "the paper's optional optimisations (P:364-377), off on the headline path (DESIGN R17); "
                   "parity: tests/test_gpu_fullsize.py (whole problem with each step)"}
    for name, kw in (("rr_exchange", {"rr_exchange": True}), ("parent_merge", {"parent_merge": True}),
                     ("rr_exchange+parent_merge", {"rr_exchange": True, "parent_merge": True})):
        def step():
            plan = Fmm2d(z, theta=cfg.theta, p=cfg.p, leaf_target=cfg.leaf_target, real_strengths=real,
                         stream=stream, **kw)
            plan.eval(m, phi, dphi)
            return plan
        plan = None
        for _ in range(warmup):
            if plan is not None:
                plan.close()
            plan = step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            plan.close()
            plan = step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        st = plan.stats()
        plan.close()
        out[name] = {"value": cfg.n / (ms / 1e3), "unit": "points/s", "ms_per_step": ms, "steps": steps,
                     "warmup": warmup, "p2p_pairs": st.get("p2p_pairs"), "weak_pairs": st.get("weak_pairs")}
    return out


def phase_times(z, m, phi, dphi, cfg, real, stream, shard_kw):
    """Device time of each phase of one extra pass (CUDA events on the launching stream)
    and the number of this library's kernel launches in one pass."""
    import torch
    from paper_1006_2269_b200 import Fmm2d
    from paper_1006_2269_b200.fmm2d import launch_count
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n0 = launch_count()
    ev[0].record(stream)
    plan = Fmm2d(z, theta=cfg.theta, p=cfg.p, leaf_target=cfg.leaf_target, real_strengths=real, stream=stream,
                 **shard_kw)
    ev[1].record(stream)
    pt = plan.eval_timed(m, phi, dphi)
    launches = launch_count() - n0
    build_ms = ev[0].elapsed_time(ev[1])
    plan.close()
    return {"build_ms": build_ms, "launches": launches, **pt}


def end_to_end(z_np, m_np, cfg, real, stream, args, shard_kw):
    """Build + eval through the C ABI with host pinned buffers; copies inside the timing."""
    import torch
    from paper_1006_2269_b200 import Fmm2d
    zh = torch.from_numpy(z_np).pin_memory()
    mh = torch.from_numpy(m_np).pin_memory()
    ph = torch.empty(cfg.n, dtype=torch.complex128).pin_memory()
    dh = torch.empty(cfg.n, dtype=torch.complex128).pin_memory()
    kw = dict(theta=cfg.theta, p=cfg.p, leaf_target=cfg.leaf_target, real_strengths=real)
    # one GPU: two problems in flight on two streams (fmm2d_build_eval with FMM2D_ASYNC_HOST:
    # each call returns once its result copies are enqueued; the strengths' copy overlaps the
    # build, and one problem's copies overlap the other's kernels); each problem has its own
    # pinned output buffers.  Several GPUs: build, then eval on the bench stream.
    NF = E2E_IN_FLIGHT
    if not shard_kw:
        # setup (outside the timed region): grow the library's memory pool once for NF plans
        # in flight, so that no build inside the timed region maps fresh device memory
        from paper_1006_2269_b200 import reserve_pool
        free, _ = torch.cuda.mem_get_info()
        reserve_pool(int(0.6 * free))
    streams = [stream] + [torch.cuda.Stream() for _ in range(NF - 1)]
    outs = [(ph, dh)] + [(torch.empty_like(ph).pin_memory(), torch.empty_like(dh).pin_memory())
                         for _ in range(NF - 1)]
    inflight = []

    def step(k):
        if shard_kw:
            plan = Fmm2d(zh, stream=stream, **kw, **shard_kw)
            plan.eval(mh, ph, dh)
            plan.close()
            return
        o = outs[k % NF]
        plan = Fmm2d.build_eval(zh, mh, o[0], o[1], stream=streams[k % NF], async_host=True, **kw)[0]
        inflight.append(plan)
        if len(inflight) > NF - 1:
            inflight.pop(0).close()          # synchronises the oldest problem's stream

    for k in range(NF):
        step(k)
    while inflight:
        inflight.pop(0).close()
    torch.cuda.synchronize()
    steps = max(2 * NF + 2, args.steps)       # enough problems that filling / draining the pipeline is small
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for k in range(steps):
        step(k)
    for st_ in streams[1:]:                     # the end of every stream's work, on stream 0
        e_side = torch.cuda.Event()
        e_side.record(st_)
        streams[0].wait_event(e_side)
    e1.record(streams[0])
    while inflight:
        inflight.pop(0).close()
    torch.cuda.synchronize()
    out = {"ms": e0.elapsed_time(e1) / steps, "h2d": 16 * cfg.n * 2, "d2h": 16 * cfg.n * 2}
    if not shard_kw:
        # latency: one synchronous problem at a time through the same call (no overlap across calls)
        reps = 3
        e0.record(stream)
        for _ in range(reps):
            Fmm2d.build_eval(zh, mh, ph, dh, stream=stream, **kw)[0].close()
        e1.record(stream)
        torch.cuda.synchronize()
        out["single_ms"] = e0.elapsed_time(e1) / reps
    return out


if __name__ == "__main__":
    main()
