"""Benchmark: serial-EEMD sifted samples per second on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Workload (default, BASELINE.json configs[4], the 1/2/4/8-GPU scaling sweep):
serial-EEMD of 4096 variates x 4096 samples (random 4-sine mixtures + noise,
fs = 4096 Hz), serialized with D = 64 (L = 17,039,296), NR = 1000
realizations, NSTD = 0.2, MaxIter 300, sharded over the GPUs (strong scaling,
total work fixed). One step = one complete decomposition of that input: every
realization sifted, ensemble sums all-reduced over NCCL, means and residue.

A "sifted sample" is one serialized sample processed by one sift iteration
(SURVEY.md §8(d)); the count is the same on CPU and GPU because sift counts
are bit-exact. value = total sifted samples of all ranks / max-over-ranks
device time of the K timed steps. Inputs are resident in HBM for `value`;
`e2e` runs the same decomposition through the public API from pinned host
memory (H2D of the multi-signal, D2H of the (M, N, K+1) tensor).
Under torchrun (N > 1) each rank owns one GPU (NCCL over NVLink).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_BYTES_PER_SIFTED_SAMPLE = 16  # one f64 read + one f64 write of the candidate
METRIC = "serial-EEMD/CEEMDAN sifted samples/sec"  # BASELINE.json metric (the % of HBM roofline is `roofline.frac`)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload(key: str):
    from paper_2106_15319_b200 import workloads as W
    cfg = dict(W.CONFIGS[key])
    x = W.config_input(key)  # (M, N)
    return cfg, x


# ------------------------------------------------------------------ our arm

def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2106_15319_b200 as se
    from paper_2106_15319_b200 import _native as N
    from paper_2106_15319_b200.parallel import ceemdan_distributed, eemd_distributed, shard_range

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg, x = workload(args.config)
    if cfg["algo"] not in ("eemd", "ceemdan"):
        raise SystemExit("bench measures the serial-EEMD / serial-CEEMDAN configs (c2, c3, c4, c5)")
    M, Nch = x.shape
    D = cfg["D"]
    ctx = se.context(local)
    ctx.set_timing(True)
    lib = ctx.lib
    scfg = {"sd_threshold": 0.2, "max_sift_iters": cfg["max_sift_iters"], "max_imfs": cfg["max_imfs"]}
    ens = {"nstd": 0.2, "nr": cfg["nr"], "base_seed": 0}
    L = M * Nch + D * (Nch - 1)
    # serialize once on the device (inputs resident in HBM for `value`)
    x_cm = torch.from_numpy(np.ascontiguousarray(x.T)).to(dev)
    s_dev = torch.empty(L, dtype=torch.float64, device=dev)

    def concat(src, dst):
        rc = lib.semd_set_stream(ctx.ptr, C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
        ctx.check(rc)
        # host-pointer-free concatenate: device entry via serial helper kernels
        ctx.check(_concat_device(lib, ctx, src, dst, M, Nch, D))

    concat(x_cm, s_dev)
    torch.cuda.synchronize(dev)

    def step():
        return decompose_sharded(cfg, s_dev, L, scfg, ens, rank, world, ctx)

    # warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    stats_tot = {"sifted_samples": 0, "eval_ms": 0.0, "kernel_launches": 0, "solve_hazards": 0, "eval_launches": 0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        ev0.record()
        for _ in range(args.steps):
            imfs, res, st = step()
            for k in stats_tot:
                stats_tot[k] += st.get(k, 0)
        ev1.record()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms, float(stats_tot["sifted_samples"]), stats_tot["eval_ms"], float(stats_tot["kernel_launches"])],
                     dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_max, sifted_all, launches_all = float(tmax[0]), float(tsum[1]), float(tsum[3])
    else:
        ms_max, sifted_all, launches_all = ms, float(t[1]), float(t[3])
    value = sifted_all / (ms_max / 1e3)
    K = int(imfs.shape[0])
    # roofline of the dominant kernel (k_eval, the sift pass) on this rank
    eval_s = stats_tot["eval_ms"] / 1e3
    peak, peak_kind = peaks()
    achieved = ALGO_BYTES_PER_SIFTED_SAMPLE * stats_tot["sifted_samples"] / eval_s / 1e9 if eval_s > 0 else None
    traffic, traffic_note = None, None
    tf = os.path.join(ROOT, "profiles", "eval_traffic.json")
    if os.path.exists(tf):  # measured DRAM bytes of one SIFT-mode k_eval launch (ncu --set full capture)
        try:
            t = json.load(open(tf))
            traffic = t.get("traffic_bytes_per_launch")
            traffic_note = {"algorithmic_bytes_per_launch": t.get("algorithmic_bytes_per_launch"),
                            "dram_bytes_per_sifted_sample": t.get("dram_bytes_per_sifted_sample"),
                            "source": t.get("source")}
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_detail": traffic_note,
            "kernel": "k_eval (sift pass)", "eval_ms_per_step": stats_tot["eval_ms"] / args.steps,
            "algorithmic_bytes": "16 B per sifted sample (SURVEY.md §8(d))"}
    # end-to-end through the public API, host buffers, copies inside the timed region
    e2e = run_e2e(args, rank, world, local, ctx, x, cfg, scfg, ens, dev)
    out = None
    if rank == 0:
        cpu = cpu_baseline(args, x, cfg, ctx) if (world == 1 and not args.no_cpu) else None
        out = {
            "metric": METRIC, "value": value, "unit": "sifted samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "config_key": args.config, "L": L, "M": M, "N": Nch, "D": D,
                       "NR": cfg["nr"], "NSTD": 0.2, "MaxIter": cfg["max_sift_iters"], "max_imfs": cfg["max_imfs"],
                       "K": K, "parallelism": f"realization-sharded x{world} (NCCL all-reduce of ensemble sums)",
                       "l2": "working set (>= 3 x 136 MB per slot + knots + 4 GB sums) exceeds the 126 MB L2; no flush",
                       "sifted_samples_per_step": sifted_all / args.steps},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches_all), "clocks": clk.summary(),
            "solve_hazards": stats_tot["solve_hazards"],
        }
    return out


def decompose_sharded(cfg, s_dev, L, scfg, ens, rank, world, ctx):
    """One whole decomposition with this rank's realization shard: EEMD (one all-reduce at the end)
    or CEEMDAN (one all-reduce per stage). Returns (imfs, residue, this rank's engine stats)."""
    from paper_2106_15319_b200.parallel import ceemdan_distributed, eemd_distributed
    if cfg["algo"] == "ceemdan":
        imfs, res = ceemdan_distributed(s_dev, L, scfg, ens, rank, world, ctx=ctx)
        return imfs, res, ctx.stats()
    return eemd_distributed(s_dev, L, scfg, ens, rank, world, ctx=ctx, k_cap=64)


def _concat_device(lib, ctx, src, dst, M, Nch, D):
    """semd_serial_decompose's first stage on device buffers: transition weights + concatenate kernels."""
    return lib.semd_concatenate_device(ctx.ptr, C.c_void_p(src.data_ptr()), M, Nch, D, C.c_void_p(dst.data_ptr()))


def run_e2e(args, rank, world, local, ctx, x, cfg, scfg, ens, dev):
    """One decomposition per step through the public API with host buffers."""
    import torch

    from paper_2106_15319_b200.parallel import eemd_distributed

    lib = ctx.lib
    M, Nch = x.shape
    D = cfg["D"]
    L = M * Nch + D * (Nch - 1)
    host_in = torch.from_numpy(np.ascontiguousarray(x.T)).pin_memory()
    steps = max(1, args.e2e_steps)
    out_buf = {}  # pinned host result buffer, allocated once (a caller reuses its buffers)

    def one_step():
        d_in = host_in.to(dev, non_blocking=True)  # H2D of the (M, N) multi-signal
        s_dev = torch.empty(L, dtype=torch.float64, device=dev)
        ctx.check(_concat_device(lib, ctx, d_in, s_dev, M, Nch, D))
        imfs, res, st = decompose_sharded(cfg, s_dev, L, scfg, ens, rank, world, ctx)
        nbytes = 0
        if rank == 0:
            modes = torch.cat([imfs, res[None, :]], 0).contiguous()
            tensor = torch.empty((modes.shape[0], Nch, M), dtype=torch.float64, device=dev)
            ctx.check(lib.semd_deconcatenate_device(ctx.ptr, C.c_void_p(modes.data_ptr()), modes.shape[0], L, M,
                                                    Nch, D, C.c_void_p(tensor.data_ptr())))
            host_out = out_buf.get(tuple(tensor.shape))
            if host_out is None:
                out_buf.clear()
                host_out = out_buf[tuple(tensor.shape)] = torch.empty(tensor.shape, dtype=torch.float64,
                                                                       pin_memory=True)
            host_out.copy_(tensor)  # D2H of the (K+1, N, M) mode tensor
            nbytes = host_out.numel() * 8
        return st.get("sifted_samples", 0), nbytes

    one_step()  # untimed: learns the mode count and allocates the pinned result buffer
    h2d = d2h = 0
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    sifted = 0
    for _ in range(steps):
        sf, nb = one_step()
        sifted += sf
        h2d += host_in.numel() * 8
        d2h += nb
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([wall, float(sifted)], dtype=torch.float64, device=dev)
        w = t.clone()
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        wall, sifted = float(w[0]), float(t[1])
    return {"value": sifted / wall, "unit": "sifted samples/s", "h2d_bytes_per_step": h2d // steps,
            "d2h_bytes_per_step": d2h // steps, "steps": steps,
            "path": f"pinned host (M,N) -> H2D -> concatenate -> sharded {cfg['algo'].upper()} (+NCCL) -> "
                    "deconcatenate -> D2H (M,N,K+1)"}


# ------------------------------------------------------------------ CPU baselines

def _ref_or_port():
    from oracle.ffi import Oracle, Ref, build, ref_available
    if ref_available():
        return Ref(), "reference"
    build()
    return Oracle(), "port"


def cpu_sample(x, cfg, threads, count=None, scale=1):
    """count realizations (default: one per thread) of the workload on `threads` CPU threads."""
    from paper_2106_15319_b200 import workloads as W  # noqa: F401
    impl, kind = _ref_or_port()
    M, Nch = x.shape
    D = cfg["D"]
    xc = np.ascontiguousarray(x.T)
    s = impl.concatenate(xc, M, Nch, D)
    count = count or threads
    t0 = time.perf_counter()
    if cfg["algo"] == "ceemdan":  # the reference ceemdan() is sequential: one full decomposition, one thread
        impl.decompose(s, 2, iters=cfg["max_sift_iters"], imfs=cfg["max_imfs"], nstd=0.2, nr=cfg["nr"])
    elif kind == "reference":
        impl.emd_realizations(s, 0, count, threads, iters=cfg["max_sift_iters"], imfs=cfg["max_imfs"], nstd=0.2)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda m: impl.eemd_partial(s, m, m + 1, iters=cfg["max_sift_iters"], imfs=cfg["max_imfs"],
                                                    nr=cfg["nr"]), range(count)))
    return time.perf_counter() - t0, kind, s


def sifted_for(s, cfg, m_end, ctx):
    """Sifted samples of realizations [0, m_end) (CEEMDAN: the whole decomposition) from the
    parity-checked GPU engine."""
    if cfg["algo"] == "ceemdan":
        import paper_2106_15319_b200 as se
        se.decompose(s, "ceemdan", max_sift_iters=cfg["max_sift_iters"], max_imfs=cfg["max_imfs"], nr=cfg["nr"])
        return ctx.stats()["sifted_samples"]
    import paper_2106_15319_b200 as se
    from paper_2106_15319_b200 import _native as N
    lib = ctx.lib
    d_s = None
    import torch
    d_s = torch.from_numpy(s).cuda()
    sums = torch.zeros((64, s.size), dtype=torch.float64, device=d_s.device)
    k = C.c_size_t()
    ctx.check(lib.semd_eemd_partial_device(ctx.ptr, C.c_void_p(d_s.data_ptr()), s.size,
                                           C.byref(N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])),
                                           C.byref(N.EnsCfg(0.2, cfg["nr"], 0, 0)), 0, m_end,
                                           C.c_void_p(sums.data_ptr()), 64, C.byref(k)))
    return ctx.stats()["sifted_samples"]


def cpu_threads():
    return max(1, min(os.cpu_count() or 1, 64))


def cpu_baseline(args, x, cfg, ctx):
    T = cpu_threads()
    if cfg["algo"] == "ceemdan":
        wall, kind, s = cpu_sample(x, cfg, 1)
        sifted = sifted_for(s, cfg, cfg["nr"], ctx)
        return {"value": sifted / wall, "unit": "sifted samples/s", "cores": 1, "kind": kind,
                "sample": f"the whole decomposition by the reference ceemdan() (sequential), wall {wall:.1f} s"}
    wall, kind, s = cpu_sample(x, cfg, T)
    sifted = sifted_for(s, cfg, T, ctx)
    return {"value": sifted / wall, "unit": "sifted samples/s", "cores": T, "kind": kind,
            "sample": f"{T} realizations (m=0..{T - 1}) of the same workload, one per thread, reference emd() each "
                      f"(eemd()'s per-realization work without its NR x K x L store); sifted count from the "
                      f"parity-checked GPU run of the same realizations; wall {wall:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on this box's host cores."""
    if rank != 0:
        return None
    cfg, x = workload(args.config)
    T = cpu_threads()
    import paper_2106_15319_b200 as se
    ctx = se.context(0)
    # warm-up: a short run on 1/16 of the realizations' length (page-in, thread start)
    for _ in range(args.warmup):
        cpu_sample(x[: max(64, x.shape[0] // 16)], cfg, T, count=T)
    total_wall, kind, s = 0.0, None, None
    for _ in range(args.steps):
        w, kind, s = cpu_sample(x, cfg, T)
        total_wall += w
    sifted = sifted_for(s, cfg, T, ctx) * args.steps
    value = sifted / total_wall
    if cfg["algo"] == "ceemdan":
        T = 1  # the reference ceemdan() is sequential
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "sifted samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "config_key": args.config,
                       "sample": f"each step = {T} realizations on {T} host threads"},
            "cpu_baseline": {"value": value, "unit": "sifted samples/s", "cores": T, "kind": kind,
                             "sample": f"{T} realizations per step, one per thread (reference emd() per realization)"},
            "e2e": {"value": value, "unit": "sifted samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = run_ours(args, rank, world, local)
    if out is not None:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
