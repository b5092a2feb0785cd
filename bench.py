#!/usr/bin/env python
"""Benchmark of the GPAIR hot path: one step = one full IR iteration
(gpair_iterate: NPC -> forward -> [allreduce] -> residual + loss -> adjoint
-> fused Adam update) on BASELINE.json's headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL): kernels are
sharded by contiguous z-slabs, the only collective is the all-reduce of the
partial signals inside gpair_iterate.  Rank 0 prints ONE JSON line.
The metric is BASELINE.json's: kernel-sensor pair evaluations per second of
the whole job (2 M N_d per iteration: forward + adjoint), and ms per iteration.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kernel-sensor pair evals/s; ms per fwd+adjoint IR iteration at 8.4M kernels"
UNIT = "pair-evals/s"
# roofline of the exact operator: 16 pair-samples / clk / SM = the
# shared-memory pipe's 128 B / clk / SM over the 8 B each pair-sample moves in both kernels
# (forward: 4-B load + 4-B store of the lane's accumulator; adjoint: one 8-B load of the lane's
# fp64 residual column) = SURVEY 8d's SFU rate of one exp per pair-sample (16 MUFU / clk / SM)
PAIR_SAMPLES_PER_CLK_SM = 16
ISSUE_PER_CLK_SM = 4  # warp instructions / clk / SM (4 SMSPs)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg4")
    p.add_argument("--op", default="exact", choices=["exact", "assa"],
                   help="exact: Eq. 7 windows (north_star); assa: the paper's ASSA operator (row f1)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--lam", type=float, default=0.0,
                   help="lambda of Eq. 23: adds R_VCR (beta 0.5) to every iteration; at N > 1 z-slab halo exchange")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU oracle sample time")
    return p.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU oracle
def cpu_oracle_sample(cfg, c, s, x, d, seconds):
    """Time the fp64 oracle (as it stands) on exact row/column subsets of the
    workload; returns (pair-evals/s, cores, description)."""
    import oracle

    op = cfg.op_kwargs()
    adj = {k: v for k, v in op.items() if k != "n_samples"}
    M, Nd = c.shape[1], s.shape[1]
    cores = oracle.threads()
    # calibrate on one row per core (the oracle parallelises over sensor rows)
    t = time.perf_counter()
    oracle.forward(c, x, s, rows=np.arange(min(cores, Nd), dtype=np.int32), **op)
    t1 = max(time.perf_counter() - t, 1e-3)  # time for `cores` rows in parallel
    n_rows = int(max(1, min(Nd, cores * round(0.5 * seconds / t1))))
    rows = np.linspace(0, Nd - 1, n_rows).astype(np.int32)
    t = time.perf_counter()
    oracle.forward(c, x, s, rows=rows, **op)
    tf = time.perf_counter() - t
    n_cols = int(max(32, min(M, n_rows * M // Nd)))
    cols = np.linspace(0, M - 1, n_cols).astype(np.int64)
    t = time.perf_counter()
    oracle.adjoint(c, d, s, cols=cols, **adj)
    ta = time.perf_counter() - t
    pairs = n_rows * M + n_cols * Nd
    rate = pairs / (tf + ta)
    desc = (f"oracle forward on {n_rows} of {Nd} sensor rows (all {M} kernels) + adjoint on {n_cols} of {M} "
            f"kernel columns (all {Nd} sensors): {pairs} pairs in {tf + ta:.1f} s")
    return rate, cores, desc


def cpu_model():
    try:
        out = subprocess.check_output(["lscpu"], text=True)
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ----------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the fp64 oracle (this tier's reference arm), timed as
    it stands on the host cores, each step a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2602_03893_b200 import inputs

    cfg = inputs.CONFIGS[args.config]
    c, s = cfg.centers(), cfg.sensors()
    x = inputs.dense_amplitudes(cfg.M)
    d = inputs.residual(cfg.n_sensors, cfg.n_samples)
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    rates, desc, cores = [], "", 1
    for i in range(args.warmup + args.steps):
        r, cores, desc = cpu_oracle_sample(cfg, c, s, x, d, budget)
        if i >= args.warmup:
            rates.append(r)
    rate = float(np.mean(rates))
    pairs_iter = 2.0 * cfg.M * cfg.n_sensors
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * pairs_iter / rate,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "kernels": cfg.M, "sensors": cfg.n_sensors,
                                        "samples": cfg.n_samples, "note": "ms_per_step extrapolated from the sample rate"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                         "cpu": cpu_model()},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2602_03893_b200 import build, gpair, inputs
    from paper_2602_03893_b200.shard import kernel_shard, max_over_ranks, nccl_bootstrap, slab_shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        build.build()
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
        comm = nccl_bootstrap(dist, rank, world, gpair.nccl_unique_id, gpair.nccl_comm_init)

    cfg = inputs.CONFIGS[args.config]
    c_all = cfg.centers()
    s = cfg.sensors()
    M = cfg.M
    lo, hi = kernel_shard(M, world, rank)  # contiguous z-slab shard
    vcr_kw = {}
    if args.lam > 0:  # whole z planes per rank, the layout R_VCR's halo exchange assumes
        P = cfg.grid[0] * cfg.grid[1]
        z0, nzr = slab_shard(cfg.grid, world, rank)
        lo, hi = z0 * P, (z0 + nzr) * P
        vcr_kw = dict(lam=args.lam, beta=0.5, eps_reg=1e-8, grid=tuple(cfg.grid), z0=z0)
    c = np.ascontiguousarray(c_all[:, lo:hi])
    Ml = hi - lo
    ctx = gpair.Context(torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev), sigma=cfg.sig, v=cfg.v,
                        fs=cfg.fs, n_samples=cfg.n_samples, t0=cfg.t0, k=cfg.k, rank=rank, world=world,
                        nccl_comm=comm, assa=(args.op == "assa"))
    if vcr_kw:  # agree on the slab layout once, before any timed collective (every rank)
        ctx.vcr_prepare(vcr_kw["grid"], vcr_kw["z0"])
    info = ctx.info()
    pair_samples_local = ctx.count_pair_samples()
    # measured data b: forward of the vessel phantom (a workload input only)
    phantom = inputs.vessel_phantom(*cfg.grid)
    b = ctx.forward(torch.from_numpy(np.ascontiguousarray(phantom[lo:hi])).to(dev))
    z = torch.zeros(Ml, device=dev)
    m = torch.zeros_like(z)
    v = torch.zeros_like(z)
    loss = torch.zeros(1, device=dev)
    eta = dict(eta_min=1e-4, eta_max=0.1, T0=50, Tmult=1)
    step = [0]

    def one_iter():
        t = step[0]
        ctx.iterate(z, m, v, b, lr=gpair.cawr_lr(t, **eta), step=t + 1, loss_out=loss, **vcr_kw)
        step[0] += 1

    for _ in range(args.warmup):
        one_iter()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile_enable(True)
    with ClockSampler(local) as clk:
        e0.record(st)
        for _ in range(args.steps):
            one_iter()
        e1.record(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    n_kernels_timed = ctx.profile_kernels()  # library kernel launches inside the timed region
    ctx.profile_enable(False)
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        ms = max_over_ranks(dist, ms, dev)
    pairs_iter = 2.0 * M * cfg.n_sensors  # whole job: forward + adjoint pairs
    value = pairs_iter / (ms * 1e-3)

    # ---- e2e through the public API with host buffers (pinned), per step:
    # h2d of b, one gpair_iterate, d2h of the loss.
    b_host = b.cpu().pin_memory()
    loss_host = torch.zeros(1).pin_memory()
    b_dev = torch.empty_like(b)
    for _ in range(2):
        b_dev.copy_(b_host, non_blocking=True)
        one_iter()
        loss_host.copy_(loss, non_blocking=True)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        b_dev.copy_(b_host, non_blocking=True)
        t = step[0]
        ctx.iterate(z, m, v, b_dev, lr=gpair.cawr_lr(t, **eta), step=t + 1, loss_out=loss, **vcr_kw)
        step[0] += 1
        loss_host.copy_(loss, non_blocking=True)
        torch.cuda.synchronize()
        _ = float(loss_host[0])
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        e2e_s = max_over_ranks(dist, e2e_s, dev)

    # ---- roofline of the dominant kernel (forward or adjoint) on this rank, and of both
    # per-step totals: with the sensor-group pipeline the forward is 4 equal launches per step
    fwd_ms, fwd_n = prof["forward"]
    adj_ms, adj_n = prof["adjoint"]
    dom = "forward" if fwd_ms >= adj_ms else "adjoint"
    dom_ms = (fwd_ms if dom == "forward" else adj_ms) / args.steps
    dom_launches = (fwd_n if dom == "forward" else adj_n) / args.steps
    clocks = clk.summary()
    f_max = (clocks["sm_max_mhz"] or 1965) * 1e6
    f_meas = (clocks["sm_mhz"] or clocks["sm_max_mhz"] or 1965) * 1e6
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    side = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            side = json.load(open(tpath)).get(("assa_" if args.op == "assa" else "") + args.config, {})
        except Exception:
            side = {}
    names = {"forward": "k_assa_forward" if args.op == "assa" else "k_forward",
             "adjoint": {0: "k_assa_adjoint" if args.op == "assa" else "k_adjoint", 1: "k_adjoint_t",
                         2: "k_adjoint_lcf", 3: "k_adjoint_sl", 4: "k_adjoint_mp"}.get(info["adj_kernel"], "adjoint")}
    if args.op == "exact":
        # units: in-window pair-samples, counted on the GPU for this context
        units, unit, bound = pair_samples_local, "Gpair-samples/s", "alu"
        peak_of = lambda f: n_sm * PAIR_SAMPLES_PER_CLK_SM * f  # noqa: E731
        peak_def = (f"{n_sm} SMs x {PAIR_SAMPLES_PER_CLK_SM} pair-samples/clk x {f_max / 1e6:.0f} MHz: 8 B of shared "
                    "memory per pair-sample (forward 4-B load + 4-B store of the accumulator column, adjoint one 8-B "
                    "load of the fp64 residual column) at 128 B/clk/SM = SURVEY 8d's one SFU exp per pair-sample; "
                    "DESIGN.md section 6")
    else:
        # ASSA (row f1): units = impulses (pairs); issue-bound: 4 warp instructions / clk / SM over the
        # kernel's executed instructions per impulse (ncu, profiles/ncu_traffic.json)
        units, unit, bound = M * cfg.n_sensors, "Gpairs/s", "issue"
        ipp = side.get("instr_per_pair", {}).get(dom)
        peak_of = (lambda f: n_sm * ISSUE_PER_CLK_SM * 32 * f / ipp) if ipp else None  # noqa: E731
        peak_def = (f"{n_sm} SMs x 4 warp-instr/clk x 32 lanes x {f_max / 1e6:.0f} MHz / {ipp} executed instructions "
                    "per impulse (ncu, cfg4): the issue bound of the kernel as built; DESIGN.md section 8b")
    per_kernel = {}
    for key, (tot_ms, n) in (("forward", prof["forward"]), ("adjoint", prof["adjoint"])):
        if not n:
            continue
        k_ms = tot_ms / args.steps
        ach = units / (k_ms * 1e-3)
        if args.op == "exact":
            kpeak = peak_of(f_max)
        else:
            kipp = side.get("instr_per_pair", {}).get(key)
            kpeak = n_sm * ISSUE_PER_CLK_SM * 32 * f_max / kipp if kipp else None
        per_kernel[names[key]] = {"ms": k_ms, "achieved": ach / 1e9, "frac": (ach / kpeak) if kpeak else None}
        if key == "adjoint" and info["adj_kernel"] == 4 and args.op == "exact":
            # the moment-polynomial adjoint reads one staged moment row per pair (no per-sample work,
            # so its pair-sample rate exceeds the per-sample roofline above): its own bound is the
            # shared-memory pipe at one staged moment row per pair (gpair_info.adj_row_bytes: 32 or
            # 48 B), 128 B / clk / SM; the launch also holds the moment prep and the group gather
            #
            row_b = info["adj_row_bytes"]
            pairs = Ml * cfg.n_sensors  # this rank's kernel shard
            own_peak = n_sm * 128.0 / row_b * f_max
            per_kernel[names[key]]["own_roofline"] = {
                "bound": "smem", "unit": "Gpairs/s", "achieved": pairs / (k_ms * 1e-3) / 1e9,
                "peak": own_peak / 1e9, "frac": pairs / (k_ms * 1e-3) / own_peak,
                "peak_def": f"{n_sm} SMs x 128 B/clk / {row_b} B per pair x {f_max / 1e6:.0f} MHz"}
    achieved = units / (dom_ms * 1e-3)
    peak = peak_of(f_max) if peak_of else None
    roof = {"bound": bound, "kernel": names[dom], "achieved": achieved / 1e9,
            "peak": peak / 1e9 if peak else None, "unit": unit, "frac": achieved / peak if peak else None,
            "traffic": side.get(dom), "frac_at_measured_clock": (achieved / peak_of(f_meas)) if peak_of else None,
            "peak_def": peak_def, "units_per_step": units, "dominant_launches_per_step": dom_launches,
            "per_kernel": per_kernel,
            "kernel_ms": {k: (v[0] / args.steps) for k, v in prof.items() if v[1]},
            "share_of_step": {k: (v[0] / args.steps) / ms for k, v in prof.items() if v[1]}}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, "operator": args.op, "kernels": M, "sensors": cfg.n_sensors, "samples": cfg.n_samples,
                   "array": cfg.array, "fs_hz": cfg.fs, "sigma_m": cfg.sig, "k": cfg.k,
                   "step": "gpair_iterate (NPC + forward + residual/loss + adjoint + Adam)"
                           + (f" + lam {args.lam:g} R_VCR (beta 0.5)" if args.lam > 0 else ""),
                   "parallelism": f"kernel-sharded x{world}" if world > 1 else "single GPU",
                   "l2": f"working set {info['workspace_bytes'] / 2**20:.0f} MiB > 126 MB L2 (no flush needed)",
                   "layout": {k: info[k] for k in ("fwd_regions", "fwd_window", "adj_regions", "adj_window", "wmax")}},
        "roofline": roof,
        "e2e": {"value": pairs_iter / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
                "h2d_bytes_per_step": int(b.numel() * 4), "d2h_bytes_per_step": 4},
        "gpu_launches": int(n_kernels_timed),
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        d = inputs.residual(cfg.n_sensors, cfg.n_samples)
        x = inputs.dense_amplitudes(cfg.M)
        rate, cores, desc = cpu_oracle_sample(cfg, c_all, s, x, d, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                                "cpu": cpu_model(), "ms_per_iter_extrapolated": 1e3 * pairs_iter / rate}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        gpair.nccl_comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
