"""Benchmark: serial-EEMD sifted samples per second on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Workload (default, BASELINE.json configs[4], the 1/2/4/8-GPU scaling sweep):
serial-EEMD of 4096 variates x 4096 samples (random 4-sine mixtures + noise,
fs = 4096 Hz), serialized with D = 64 (L = 17,039,296), NR = 1000
realizations, NSTD = 0.2, MaxIter 300, sharded over the GPUs (strong scaling,
total work fixed). One step = one complete decomposition of that input: every
realization sifted, ensemble sums reduced over NCCL, means and residue.

A "sifted sample" is one serialized sample processed by one sift iteration
(SURVEY.md §8(d)); the count is the same on CPU and GPU because sift counts
are bit-exact. value = total sifted samples of all ranks / max-over-ranks
device time (CUDA events on the engine stream) of the K timed steps. Inputs
are resident in HBM for `value`; `e2e` runs the same decomposition through the
public host-pointer C ABI (semd_serial_decompose) from pinned host memory: H2D
of the (M, N) multi-signal, concatenate, sharded EEMD (+NCCL), deconcatenate,
D2H of the (M, N, K+1) tensor.

Under torchrun (N > 1) each rank owns one GPU; the ranks' engine contexts are
joined by an NCCL communicator inside the C ABI (semd_comm_*). No torch on
any path of this file. The CPU legs (cpu_baseline, --impl reference) run the
reference compiled from its own sources (oracle/_ref) and count sifted samples
on the CPU with the reference's own extract_imf.
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
ALGO_ID = {"emd": 0, "eemd": 1, "ceemdan": 2}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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
        if os.environ.get("SEMD_BENCH_NO_SMI"):  # diagnosis: no sampler process during the timed region
            return self
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


# ------------------------------------------------------------------ our arm (C ABI only)

class Dev:
    """A device (or pinned host) buffer owned through the C ABI."""

    def __init__(self, ctx, nbytes: int, pinned_host: bool = False):
        self.ctx, self.host = ctx, pinned_host
        p = C.c_void_p()
        ctx.run("semd_host_alloc" if pinned_host else "semd_device_alloc", int(nbytes), C.byref(p))
        self.ptr, self.nbytes = p, int(nbytes)

    def free(self):
        if self.ptr:
            self.ctx.run("semd_host_free" if self.host else "semd_device_free", self.ptr)
            self.ptr = None


def _stats(ctx) -> dict:
    return ctx.stats()


def run_ours(args, rank, world, local):
    import paper_2106_15319_b200 as se
    from paper_2106_15319_b200 import _native as N
    from paper_2106_15319_b200.parallel import init_comm

    cfg, x = workload(args.config)
    if cfg["algo"] not in ("eemd", "ceemdan"):
        raise SystemExit("bench measures the serial-EEMD / serial-CEEMDAN configs (c2, c3, c4, c5)")
    ctx = se.context(local)
    init_comm(ctx, rank, world, root=0)  # EEMD sums reduced to rank 0; CEEMDAN stages all-reduced
    ctx.set_timing(True)
    M, Nch = x.shape
    D = cfg["D"]
    L = M * Nch + D * (Nch - 1)
    algo = ALGO_ID[cfg["algo"]]
    scfg = N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])
    ens = N.EnsCfg(0.2, cfg["nr"], 0, 0)
    xc = np.ascontiguousarray(x.T)  # channel-contiguous MultiSignal (types.hpp:61-62)
    # inputs resident in HBM for `value`: the multi-signal and its serialization
    d_x = Dev(ctx, xc.nbytes)
    ctx.run("semd_memcpy", d_x.ptr, xc.ctypes.data_as(C.c_void_p), xc.nbytes)
    d_s = Dev(ctx, L * 8)
    ctx.run("semd_concatenate_device", d_x.ptr, M, Nch, D, d_s.ptr)
    k_cap = 32
    d_imfs, d_res = Dev(ctx, k_cap * L * 8), Dev(ctx, L * 8)
    kout = C.c_size_t()

    def step():
        ctx.run("semd_decompose_device", algo, d_s.ptr, L, C.byref(scfg), C.byref(ens), d_imfs.ptr, k_cap,
                C.byref(kout), d_res.ptr)
        return _stats(ctx)

    def barrier():
        ctx.comm_allreduce([0.0])

    for _ in range(args.warmup):
        step()
    keys = ("sifted_samples", "eval_ms", "kernel_launches", "solve_hazards", "eval_launches")
    tot = dict.fromkeys(keys, 0)
    with ClockSampler(local) as clk:
        barrier()
        ctx.run("semd_timer_start")
        for _ in range(args.steps):
            st = step()
            for k in keys:
                tot[k] += st[k]
        ms = C.c_double()
        ctx.run("semd_timer_stop", C.byref(ms))
        barrier()
    ms_max = float(ctx.comm_allreduce([ms.value], "max")[0])
    sums = ctx.comm_allreduce([float(tot["sifted_samples"]), float(tot["kernel_launches"]),
                               float(tot["solve_hazards"])], "sum")
    sifted_all, launches_all, hazards_all = float(sums[0]), int(sums[1]), int(sums[2])
    value = sifted_all / (ms_max / 1e3)
    K = int(kout.value)
    peak, peak_kind = peaks()
    # BASELINE.md roofline: 16 B x sifted samples / wall / peak, per GPU, over the whole step
    achieved = ALGO_BYTES_PER_SIFTED_SAMPLE * sifted_all / world / (ms_max / 1e3) / 1e9
    eval_s = tot["eval_ms"] / 1e3
    eval_ach = ALGO_BYTES_PER_SIFTED_SAMPLE * tot["sifted_samples"] / eval_s / 1e9 if eval_s > 0 else None
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "r02", f"traffic_{args.config}.json")
    if os.path.exists(tf):  # dram bytes of the dominant kernel from an ncu --set full capture of this config
        try:
            t = json.load(open(tf))
            traffic, traffic_src = t.get("traffic_bytes_per_launch"), t
        except Exception:
            traffic = None
    resident = _stats(ctx)["resident_jobs"] > 0  # short signals: the resident engine ran the step
    dom_name = ("k_res_ceemdan (the whole CEEMDAN: one persistent CTA per realization task, candidate and "
                "segment tables in shared memory)" if cfg["algo"] == "ceemdan" else
                "k_resident (one persistent CTA per realization, candidate and segment tables in shared memory)") \
        if resident else "k_eval (sift pass: envelopes, mean, SD sums, next extrema detection)"
    dom_timing = ("CUDA events around the resident-engine launch on the engine stream" if resident else
                  "device time of every k_eval launch (%globaltimer span, first CTA start to last CTA end)")
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "scope": "whole step: 16 B x sifted samples / device time of the step / N GPUs (BASELINE.md)",
            "dominant_kernel": {
                "kernel": dom_name,
                "achieved": eval_ach, "frac": (eval_ach / peak) if eval_ach else None,
                "ms_per_step": tot["eval_ms"] / args.steps,
                "share_of_step": (tot["eval_ms"] / args.steps) / (ms.value / args.steps) if ms.value else None,
                "timing": dom_timing,
                "launches_per_step": tot["eval_launches"] / args.steps},
            "traffic_detail": traffic_src,
            "algorithmic_bytes": "16 B per sifted sample (SURVEY.md §8(d))"}
    e2e = run_e2e(args, rank, world, ctx, xc, cfg, algo, scfg, ens)
    for b in (d_x, d_s, d_imfs, d_res):
        b.free()
    out = None
    if rank == 0:
        cpu = cpu_baseline(args, x, cfg, ctx) if (world == 1 and not args.no_cpu) else None
        out = {
            "metric": METRIC, "value": value, "unit": "sifted samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "config_key": args.config, "L": L, "M": M, "N": Nch, "D": D,
                       "NR": cfg["nr"], "NSTD": 0.2, "MaxIter": cfg["max_sift_iters"], "max_imfs": cfg["max_imfs"],
                       "K": K, "parallelism": f"realization-sharded x{world} (NCCL reduce of ensemble sums "
                                              "inside the C ABI)" if world > 1 else "single GPU",
                       "l2": "working set (>= 3 x 136 MB per slot + knots + 4 GB sums) exceeds the 126 MB L2; "
                             "no flush" if args.config in ("c4", "c5") else "small signal (L2-resident); "
                                                                              "latency-bound config",
                       "sifted_samples_per_step": sifted_all / args.steps},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_all, "clocks": clk.summary(), "solve_hazards": hazards_all,
        }
    return out


def run_e2e(args, rank, world, ctx, xc, cfg, algo, scfg, ens):
    """The public host-pointer C ABI (semd_serial_decompose): pinned host (N, M) multi-signal in,
    pinned host (K+1, N, M) ImfTensor out, copies inside the timed region."""
    N_, M = xc.shape
    D = cfg["D"]
    k_cap = 33
    h_in = Dev(ctx, xc.nbytes, pinned_host=True)
    C.memmove(h_in.ptr, xc.ctypes.data, xc.nbytes)
    h_out = Dev(ctx, k_cap * N_ * M * 8, pinned_host=True)
    mo = C.c_size_t()

    def one():
        ctx.run("semd_serial_decompose", algo, C.cast(h_in.ptr, C.POINTER(C.c_double)), M, N_, D, C.byref(scfg),
                C.byref(ens), C.cast(h_out.ptr, C.POINTER(C.c_double)), k_cap, C.byref(mo), None)
        return ctx.stats()["sifted_samples"]

    one()  # untimed: first-call allocations
    steps = max(1, args.e2e_steps)
    ctx.comm_allreduce([0.0])
    t0 = time.perf_counter()
    sifted = 0
    for _ in range(steps):
        sifted += one()
    wall = time.perf_counter() - t0
    ctx.comm_allreduce([0.0])
    wall = float(ctx.comm_allreduce([wall], "max")[0])
    sifted = float(ctx.comm_allreduce([float(sifted)], "sum")[0])
    d2h = int(mo.value) * N_ * M * 8  # the ImfTensor, on the rank that holds the result
    h_in.free()
    h_out.free()
    return {"value": sifted / wall, "unit": "sifted samples/s", "h2d_bytes_per_step": xc.nbytes * world,
            "d2h_bytes_per_step": d2h, "steps": steps, "timing": "host wall clock around the ABI call, max over ranks",
            "path": "semd_serial_decompose: pinned host (M,N) -> H2D -> concatenate -> "
                    f"{cfg['algo'].upper()}{' (+NCCL)' if world > 1 else ''} -> deconcatenate -> D2H (M,N,K+1)"}


# ------------------------------------------------------------------ CPU baselines (reference only)

def cpu_threads():
    return max(1, min(os.cpu_count() or 1, 64))


def _ref():
    from oracle.ffi import Oracle, Ref, build, ref_available
    if ref_available():
        return Ref(), "reference"
    build()
    return Oracle(), "port"


def ceemdan_sifted(trace, n: int) -> int:
    """n x (find_extrema calls of the CEEMDAN replay that led to a subtraction): the reference's
    own extract_imf loop (emd.cpp:131-151) subtracts iff both envelopes exist."""
    ok = (trace["task"] != 3) & (trace["n_max"] >= 2) & (trace["n_min"] >= 2)
    return int(n) * int(ok.sum())


class CpuSample:
    """A bounded sample of the workload on the reference CPU implementation, with its sifted-sample
    count computed on the CPU (outside any timed region) by the reference's own extract_imf."""

    def __init__(self, x, cfg, threads):
        self.impl, self.kind = _ref()
        M, Nch = x.shape
        self.s = self.impl.concatenate(np.ascontiguousarray(x.T), M, Nch, cfg["D"])
        self.cfg, self.T = cfg, threads
        it, im = cfg["max_sift_iters"], cfg["max_imfs"]
        if cfg["algo"] == "ceemdan":  # the reference ceemdan() is sequential: the whole decomposition, one thread
            self.T = 1
            if self.kind == "reference":
                _, _, tr = self.impl.ceemdan_traced(self.s, iters=it, imfs=im, nr=cfg["nr"])
                self.sifted = ceemdan_sifted(tr, self.s.size)
            else:
                _, _, _, tr = self.impl.decompose(self.s, 2, iters=it, imfs=im, nr=cfg["nr"], trace_cap=1 << 22)
                self.sifted = ceemdan_sifted(tr, self.s.size)
            self.per_m = None
            self.desc = "the whole decomposition by the reference ceemdan() (sequential, one thread)"
        else:
            if self.kind == "reference":
                self.sifted, self.per_m = self.impl.realization_sifts(self.s, 0, self.T, self.T, iters=it, imfs=im)
            else:
                raise RuntimeError("oracle/_ref (the reference built from its sources) is required for EEMD baselines")
            self.desc = (f"{self.T} realizations (m=0..{self.T - 1}) of the same workload, one per host thread, each "
                         "the reference emd() of x + beta*white_noise(derive_seed(0, m)) (eemd()'s per-realization "
                         "work without its NR x K x L store)")

    def run(self, x_short=None) -> float:
        it, im = self.cfg["max_sift_iters"], self.cfg["max_imfs"]
        s = self.s if x_short is None else x_short
        t0 = time.perf_counter()
        if self.cfg["algo"] == "ceemdan":
            self.impl.decompose(s, 2, iters=it, imfs=im, nr=self.cfg["nr"])
        else:
            self.impl.emd_realizations(s, 0, self.T, self.T, iters=it, imfs=im)
        return time.perf_counter() - t0


def gpu_per_realization_sifts(s, cfg, T) -> list[int]:
    """GPU sift counts of realizations m = 0..T-1 (same beta and seeds as the NR ensemble), from the
    engine's parity trace: one record per find_extrema call; a call with both envelopes subtracts."""
    import paper_2106_15319_b200 as se
    from paper_2106_15319_b200 import _native as N
    c = se.context(0)
    cap = 400 * T
    buf = (N.TraceRec * cap)()
    tr = N.Trace(C.cast(buf, C.c_void_p), cap, 0)
    k = C.c_size_t()
    x = np.ascontiguousarray(s, dtype=np.float64)
    c.run("semd_decompose", ALGO_ID["eemd"], x.ctypes.data_as(N._dp), x.size,
          C.byref(N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])), C.byref(N.EnsCfg(0.2, T, 0, 0)),
          None, 64, C.byref(k), None, None, C.byref(tr))
    rec = np.frombuffer(C.string_at(buf, min(tr.count, cap) * C.sizeof(N.TraceRec)),
                        dtype=[("task", "<i4"), ("m", "<i4"), ("k", "<i4"), ("iter", "<i4"), ("n_max", "<u4"),
                               ("n_min", "<u4"), ("hash", "<u8")])
    ok = (rec["task"] == 0) & (rec["n_max"] >= 2) & (rec["n_min"] >= 2)
    return [int((ok & (rec["m"] == m)).sum()) for m in range(T)]


def cpu_baseline(args, x, cfg, ctx):
    T = cpu_threads()
    smp = CpuSample(x, cfg, T)
    wall = smp.run()
    out = {"value": smp.sifted / wall, "unit": "sifted samples/s", "cores": smp.T, "kind": smp.kind,
           "sample": f"{smp.desc}; sifted samples {smp.sifted} counted on the CPU by the reference's extract_imf "
                     f"(outside the timed region); wall {wall:.1f} s"}
    if smp.per_m is not None:  # free full-size parity: the GPU's per-realization sift counts must equal the CPU's
        gpu = gpu_per_realization_sifts(smp.s, cfg, smp.T)
        out["gpu_sift_counts_equal_cpu"] = bool(list(map(int, smp.per_m)) == gpu)
        out["per_realization_sifts"] = list(map(int, smp.per_m))
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation (oracle/_ref, built from its sources)
    on this box's host cores. Never loads the GPU library."""
    if rank != 0:
        return None
    cfg, x = workload(args.config)
    T = cpu_threads()
    smp = CpuSample(x, cfg, T)  # sifted-sample count on the CPU, outside the timed region
    short = smp.impl.concatenate(np.ascontiguousarray(x[: max(64, x.shape[0] // 16)].T),
                                 max(64, x.shape[0] // 16), x.shape[1], cfg["D"])
    for _ in range(args.warmup):  # page-in, thread start: the sample on 1/16 of the rows
        smp.run(short)
    total = 0.0
    for _ in range(args.steps):
        total += smp.run()
    value = smp.sifted * args.steps / total
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "sifted samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "config_key": args.config,
                       "sample": f"each step = {smp.desc}"},
            "cpu_baseline": {"value": value, "unit": "sifted samples/s", "cores": smp.T, "kind": smp.kind,
                             "sample": f"{smp.desc}; {smp.sifted} sifted samples per step, counted on the CPU"},
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
    out = run_reference(args, rank, world) if args.impl == "reference" else run_ours(args, rank, world, local)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
