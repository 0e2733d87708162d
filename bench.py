#!/usr/bin/env python
"""Benchmark: multi-LoRA delta tokens/s (InfiniLoRA LoRA-Server hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

One *step* = one pass of the whole hot path over one batch: a1 segmentation
(lora_plan_build) + a2-a4 for every slot of the unit of work (gate, up, down
of one Mixtral MoE layer, multi-slot apply).  Default workload: BASELINE.json
config 5 (mixtral_sharded: 2048 adapters, 4096 tokens -> 8192 rows), the
config the metric is quoted on at 1/2/4/8 GPUs; it fits one B200 (116 GB of
weights).  N=1 runs the unsharded server; N>1 runs the adapter-sharded server
(owner(a) = (a - h) mod N for a >= h, the h hottest adapters replicated on
every rank; NCCL send/recv over NVLink), launched by torchrun.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import dataclasses
import faulthandler
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import lora_inputs as li  # noqa: E402

METRIC = "multi-LoRA delta tokens/s at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "tokens/s"
NOMINAL_HBM_GBS = 8000.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1660.1)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# algorithmic bytes
# ---------------------------------------------------------------------------
def algorithmic(cfg: li.Config, batch: li.Batch, slots, small_max: int = 8):
    """Algorithmic bytes per step, split by kernel.

    Each touched unit's A and B are read once, each valid row's x once per
    distinct x buffer (slots sharing x -- gate/up, q/k/v -- need it once),
    its y read + written once; a segment of more than `small_max` rows
    runs on the tcgen05 kernels (rank 16 / 32 / 64 / 128, 128-multiple
    widths, the large segments holding at least LORA_TC_MIN_ROWS rows
    together: 256, 2048 at r = 16), else on the CUDA-core kernels -- the same
    dispatch rule the library applies."""
    a = batch.adapter_ids.astype(np.int64)
    valid = a >= 0
    T, Tv = batch.n_rows, int(valid.sum())
    ysz = 4 if cfg.y_dtype == "fp32" else 2
    r = cfg.rank
    tc_ok = r in (8, 16, 32, 64, 128) and small_max >= 0 and all(s.h_in % 128 == 0 and s.h_out % 128 == 0
                                                               for s in cfg.slots)
    if tc_ok:  # the segmenter's device-side rule over the plan (one plan per apply)
        E0 = cfg.slots[slots[0]].n_experts
        _, c0 = np.unique(a[valid] * E0 + batch.expert_ids[valid], return_counts=True)
        min_rows = int(os.environ.get("LORA_TC_MIN_ROWS", 2048 if r <= 16 else 256))
        tc_ok = int(c0[c0 > small_max].sum()) >= min_rows
    out = {"segment": T * 8, "simt_shrink": 0, "simt_expand": 0, "tc05_shrink": 0, "tc05_expand": 0,
           "flops": 0, "units": {}}
    seen_x = set()
    for i in slots:
        sl = cfg.slots[i]
        _, cnt = np.unique(a[valid] * sl.n_experts + batch.expert_ids[valid], return_counts=True)
        out["units"][sl.name] = int(cnt.size)
        big = (cnt > small_max) if tc_ok else np.zeros(cnt.size, bool)
        # x is an input of the step: slots sharing it (gate/up, q/k/v) need it read once
        x_once = sl.xbuf not in seen_x
        seen_x.add(sl.xbuf)
        for path, m in (("simt", ~big), ("tc05", big)):
            U, rows = int(m.sum()), int(cnt[m].sum())
            out[path + "_shrink"] += U * sl.h_in * r * 2 + (rows * sl.h_in * 2 if x_once else 0)
            out[path + "_expand"] += U * sl.h_out * r * 2 + rows * sl.h_out * 2 * ysz
        out["flops"] += 2 * Tv * r * (sl.h_in + sl.h_out)
    out["shrink"] = out["simt_shrink"] + out["tc05_shrink"]
    out["expand"] = out["simt_expand"] + out["tc05_expand"]
    out["total"] = out["segment"] + out["shrink"] + out["expand"]
    out["rows_valid"] = Tv
    return out


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for l in self.lines:
            p = [v.strip() for v in l.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N=1 only) and the --impl reference arm
# ---------------------------------------------------------------------------
def oracle_sample(cfg, batch, slots, n_tokens):
    """Prepared oracle inputs for the first n_tokens tokens (all slots)."""
    from oracle import oracle as orc
    rows = np.arange(n_tokens * batch.top_k)
    return [orc.prepare_slot(cfg, i, batch, rows) for i in slots]


def oracle_time(prepared, n_threads: int = 0):
    from oracle import oracle as orc
    t0 = time.perf_counter()
    for (x, uor, sor, A, B, y) in prepared:
        orc.lora_apply_rows(x, uor, sor, A, B, y.copy(), n_threads=n_threads)
    return time.perf_counter() - t0


def cpu_model() -> str:
    """The host CPU's model name (lscpu / /proc/cpuinfo), for the oracle's timing."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, batch, slots, budget_s=10.0):
    """Grow the token sample until one oracle pass costs ~budget_s (or the batch ends)."""
    from oracle import oracle as orc
    n = 16
    best = None
    while True:
        prep = oracle_sample(cfg, batch, slots, n)
        dt = oracle_time(prep)
        best = (n, dt)
        if dt >= budget_s / 4 or n >= batch.n_tokens:
            break
        n = min(batch.n_tokens, max(n * 2, int(n * (budget_s / 4) / max(dt, 1e-3))))
    n, dt = best
    # the same oracle on one thread (--threads 1 and --threads nproc)
    n1 = max(1, min(n, int(n * 2.0 / max(dt * orc.max_threads(), 1e-3))))
    dt1 = oracle_time(prep if n1 == n else oracle_sample(cfg, batch, slots, n1), n_threads=1)
    return {"value": n / dt, "unit": UNIT, "cores": orc.max_threads(), "kind": "oracle", "cpu": cpu_model(),
            "sample": f"first {n} of {batch.n_tokens} tokens ({n * batch.top_k} rows) of the {cfg.name} batch, "
                      f"{len(slots)} slots; plain-C fp64 oracle, OpenMP over rows; input generation excluded; "
                      f"one pass = {dt:.2f} s",
            "single_thread": {"value": n1 / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"first {n1} tokens, one pass = {dt1:.2f} s"}}


def run_reference(args, cfg, batch, slots):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc
    # size one step at ~0.2 s of oracle compute
    n = 8
    while True:
        prep = oracle_sample(cfg, batch, slots, n)
        dt = oracle_time(prep)
        if dt >= 0.2 or n >= batch.n_tokens:
            break
        n = min(batch.n_tokens, n * 2)
    for _ in range(args.warmup):
        oracle_time(prep)
    times = [oracle_time(prep) for _ in range(args.steps)]
    ms = 1e3 * float(np.mean(times))
    ms_median, ms_min = 1e3 * float(np.median(times)), 1e3 * float(np.min(times))
    value = n / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_median": ms_median, "ms_min": ms_min,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "global_batch": cfg.n_tokens, "sample_tokens": n,
                       "rows": n * batch.top_k, "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": orc.max_threads(), "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": f"first {n} of {cfg.n_tokens} tokens of {cfg.name}, {len(slots)} slots, "
                                       f"input generation excluded"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm: single-GPU runner (the metric config at N=1, the secondaries, E10/E13)
# ---------------------------------------------------------------------------
class SingleRun:
    """One unsharded server + device-resident inputs of one workload; a step =
    plan build + one multi-slot apply, captured once in a CUDA graph."""

    def __init__(self, B, torch, cfg, batch, slots, dev, stream, graph=True, server=None, max_rows=0):
        self.B, self.torch, self.cfg, self.batch, self.slots = B, torch, cfg, batch, slots
        self.dev, self.stream = dev, stream
        T = self.T = batch.n_rows
        self.E = cfg.slots[slots[0]].n_experts
        self.dt = B.LORA_FP32 if cfg.y_dtype == "fp32" else B.LORA_BF16
        self.ysz = 4 if cfg.y_dtype == "fp32" else 2
        self.own_server = server is None
        if server is None:
            c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                              [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(),
                              max(T, max_rows, 1), dev.index or 0)
            server = B.lora_server_create(c)
            B.lora_server_fill_synthetic(server, cfg.seed, stream)
        self.s = server
        self.xs = {}
        for i in slots:
            sl = cfg.slots[i]
            if sl.xbuf not in self.xs:
                x = torch.empty((T, sl.h_in), dtype=torch.int16, device=dev)
                B.lora_synth_fill_rows(x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x(), 0, stream)
                self.xs[sl.xbuf] = x
        self.x_list = [self.xs[cfg.slots[i].xbuf] for i in slots]
        self.ys = []
        for i in slots:
            sl = cfg.slots[i]
            y = torch.empty((T, sl.h_out), dtype=torch.int16, device=dev)
            B.lora_synth_fill_rows(y, T, sl.h_out, cfg.seed, li.tag_of(li.KIND_Y0, i), li.shift_y0(), 0, stream)
            if self.ysz == 4:
                y = ((y.to(torch.int32) << 16).view(torch.float32)).contiguous()
            self.ys.append(y)
        self.ad = torch.from_numpy(batch.adapter_ids.copy()).to(dev)
        self.ex = torch.from_numpy(batch.expert_ids.copy()).to(dev)
        self.plan = B.lora_plan_create(self.s, max(T, 1))
        self.run = self.step
        self.graph = None
        if graph:
            # the whole step (plan build + multi-slot apply, including the fork /
            # join of the tcgen05 side stream) captured once, replayed each step
            g_stream = torch.cuda.Stream()
            g_stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(g_stream):
                self.step(g_stream)  # warm the lazy allocations outside the capture
                torch.cuda.synchronize()
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph, stream=g_stream):
                    self.step(g_stream)
            torch.cuda.current_stream().wait_stream(g_stream)
            self.run = lambda st=None: self.graph.replay()
        torch.cuda.synchronize()

    def step(self, st=None):
        B, st = self.B, (self.stream if st is None else st)
        B.lora_plan_build(self.s, self.plan, self.ad, self.ex if self.E > 1 else None, self.T, self.E, st)
        B.lora_apply_plan_multi(self.s, self.plan, self.slots, self.x_list, self.ys, self.dt, st)

    def time(self, steps, warmup):
        """Per-step device times (ms) from CUDA events on the launching stream."""
        torch = self.torch
        for _ in range(warmup):
            self.run()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        torch.cuda.synchronize()
        ev[0].record(self.stream)
        for k in range(steps):
            self.run()
            ev[k + 1].record(self.stream)
        torch.cuda.synchronize()
        return [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)], ev[0].elapsed_time(ev[-1])

    def profile(self, n):
        """Per-kernel durations: the same steps with every kernel serialised on
        the stream and a CUDA-event pair around each launch."""
        B = self.B
        B.lora_server_set_concurrent(self.s, False)
        B.lora_profile_enable(self.s, n * 32 + 16)
        for _ in range(n):
            self.step()
        self.torch.cuda.synchronize()
        prof = B.lora_profile_read(self.s)
        B.lora_profile_enable(self.s, 0)
        B.lora_server_set_concurrent(self.s, True)
        return prof

    def destroy(self):
        self.B.lora_plan_destroy(self.plan)
        if self.own_server:
            self.B.lora_server_destroy(self.s)
        self.xs, self.ys, self.x_list = {}, [], []


def kernel_table(prof, n_prof, alg):
    kern = {}
    for name, (n, tot) in prof.items():
        kern[name] = {"launches": n, "ms_per_launch": tot / n, "ms_per_step": tot / n_prof}
        b = alg.get(name)
        if b:
            kern[name]["algorithmic_GBs"] = b * n_prof / n / (tot / n * 1e-3) / 1e9
    return kern


def summarise(cfg, alg, times, total_ms, hbm_peak, prof=None, n_prof=1):
    ms = total_ms / len(times)
    gbs = alg["total"] / (ms * 1e-3) / 1e9
    out = {"ms_per_step": ms, "ms_median": float(np.median(times)), "ms_min": float(np.min(times)),
           "tokens_per_s": cfg.n_tokens / (ms * 1e-3), "rows": int(alg["rows_valid"]),
           "distinct_units": alg["units"], "algorithmic_GB": alg["total"] / 1e9, "step_GBs": gbs,
           "frac_measured": gbs / hbm_peak, "frac_nominal_8TBs": gbs / NOMINAL_HBM_GBS,
           "tflops": alg["flops"] / (ms * 1e-3) / 1e12}
    if prof is not None:
        out["kernels"] = kernel_table(prof, n_prof, alg)
    return out


def secondaries(B, torch, dev, stream, hbm_peak, steps, warmup):
    """Configs 3, 2, 4 measured in the same run (config 3 is
    the north-star >= 60 % HBM target), then E10 (batch sweep on config-3
    shapes) and E13 (the paper's kernel microbenchmark workload: 512
    adapters, batch 1024, Zipf 1.2)."""
    out = {}
    for name in ("mixtral_decode", "llama_decode", "mixtral_prefill"):
        cfg = li.CONFIGS[name]
        b = li.make_batch(cfg)
        slots = list(range(len(cfg.slots)))
        # config 3's server also serves the E10 sweep (up to 4096 tokens = 8192 rows)
        r = SingleRun(B, torch, cfg, b, slots, dev, stream, max_rows=8192 if name == "mixtral_decode" else 0)
        times, tot = r.time(steps, warmup)
        prof = r.profile(5)
        out[name] = summarise(cfg, algorithmic(cfg, b, slots), times, tot, hbm_peak, prof, 5)
        if name == "mixtral_decode":
            # E10 / E13 reuse this server (512 adapters, config-3 slots)
            srv = r.s
            r.own_server = False
            r.destroy()
            sweep = {}
            for n_tok in (64, 128, 256, 512, 1024, 2048, 4096):
                c2 = li.with_tokens(cfg, n_tok)
                b2 = li.make_batch(c2)
                if c2.n_rows > 8192:  # the server's row capacity
                    break
                r2 = SingleRun(B, torch, c2, b2, slots, dev, stream, server=srv)
                t2, tot2 = r2.time(max(5, steps // 2), 2)
                prof2 = r2.profile(3) if n_tok == 1024 else None
                sm = summarise(c2, algorithmic(c2, b2, slots), t2, tot2, hbm_peak, prof2, 3)
                r2.destroy()
                sweep[str(n_tok)] = {k: sm[k] for k in ("ms_per_step", "ms_median", "tokens_per_s", "rows",
                                                        "distinct_units", "step_GBs", "frac_measured")}
                if n_tok == 1024:
                    k = sm["kernels"]
                    sh = sum(k[n]["ms_per_step"] for n in k if n.endswith("shrink"))
                    ex = sum(k[n]["ms_per_step"] for n in k if n.endswith("expand") or n == "tc05_vreduce")
                    a2 = algorithmic(c2, b2, slots)
                    out["E13_kernel_microbench"] = {
                        "workload": "512 adapters, batch 1024 tokens (2048 rows, top-2), Zipf 1.2, Mixtral "
                                    "gate/up/down r=64 (P:790)",
                        "shrink_ms": sh, "shrink_GBs": a2["shrink"] / (sh * 1e-3) / 1e9,
                        "expand_ms": ex, "expand_GBs": a2["expand"] / (ex * 1e-3) / 1e9,
                        "kernels": k}
            B.lora_server_destroy(srv)
            out["E10_batch_sweep"] = {
                "workload": "config-3 shapes (Mixtral gate/up/down r=64, 512 adapters, Zipf 1.2, top-2); "
                            "tokens -> ms per layer (P:723: LoRA compute sub-linear in batch)",
                "points": sweep}
        else:
            r.destroy()
    # SURVEY 8d variants: uniform adapter ids (3u, Llama ~110 adapters) and the
    # 16 x 512-token prefill
    var = {}
    for name, cfg in li.VARIANTS.items():
        b = li.make_batch(cfg)
        slots = list(range(len(cfg.slots)))
        r = SingleRun(B, torch, cfg, b, slots, dev, stream)
        tv, totv = r.time(max(5, steps // 2), 2)
        profv = r.profile(3)
        sm = summarise(cfg, algorithmic(cfg, b, slots), tv, totv, hbm_peak, profv, 3)
        r.destroy()
        var[name] = {k: sm[k] for k in ("ms_per_step", "ms_median", "tokens_per_s", "rows", "step_GBs",
                                        "frac_measured", "frac_nominal_8TBs", "kernels")}
        var[name]["distinct_units"] = sum(sm["distinct_units"].values()) // max(1, len(sm["distinct_units"]))
    out["variants"] = var
    # rank sweep over the paper's range ("r typically 32-128") on config-3
    # shapes with 128 adapters (r = 64 is config 3 itself, above)
    sweep = {}
    for rk in (16, 32, 128):
        c3 = dataclasses.replace(li.CONFIGS["mixtral_decode"], name=f"mixtral_decode_r{rk}", rank=rk, n_adapters=128)
        b3 = li.make_batch(c3)
        slots = list(range(len(c3.slots)))
        r = SingleRun(B, torch, c3, b3, slots, dev, stream)
        t3, tot3 = r.time(max(5, steps // 2), 2)
        prof3 = r.profile(3)
        sm = summarise(c3, algorithmic(c3, b3, slots), t3, tot3, hbm_peak, prof3, 3)
        r.destroy()
        sweep[str(rk)] = {k: sm[k] for k in ("ms_per_step", "ms_median", "tokens_per_s", "rows", "distinct_units",
                                             "step_GBs", "frac_measured", "kernels")}
    out["rank_sweep"] = {
        "workload": "config-3 shapes (Mixtral gate/up/down, top-2, 512 tokens, Zipf 1.2) with 128 adapters at "
                    "r = 16 / 32 / 128 (P:165)",
        "points": sweep}
    # the same at prefill shapes (config 4: 8192 tokens, 16384 rows): the
    # tcgen05 chain at every rank (r = 64 is config 4 itself, above)
    sweep = {}
    for rk in (8, 16, 32, 128):
        c4 = dataclasses.replace(li.CONFIGS["mixtral_prefill"], name=f"mixtral_prefill_r{rk}", rank=rk)
        b4 = li.make_batch(c4)
        slots = list(range(len(c4.slots)))
        r = SingleRun(B, torch, c4, b4, slots, dev, stream)
        t4, tot4 = r.time(max(5, steps // 2), 2)
        prof4 = r.profile(3)
        sm = summarise(c4, algorithmic(c4, b4, slots), t4, tot4, hbm_peak, prof4, 3)
        r.destroy()
        sweep[str(rk)] = {k: sm[k] for k in ("ms_per_step", "ms_median", "tokens_per_s", "rows", "step_GBs",
                                             "frac_measured", "kernels")}
    out["prefill_rank_sweep"] = {
        "workload": "config-4 shapes (Mixtral gate/up/down, 4 x 2048-token sequences, 64 adapters, top-2) at "
                    "r = 8 / 16 / 32 / 128 (P:165); large segments on the tcgen05 chain at every rank",
        "points": sweep}
    return out


def run_ours(args, cfg, batch, slots):
    import torch
    import torch.distributed as dist

    from paper_2604_07173_b200 import binding as B

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 or args.force_sharded:
        return run_sharded(args, cfg, batch, slots)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    hbm_peak, tc_peak, peak_src = load_peaks()
    E = cfg.slots[slots[0]].n_experts

    run = SingleRun(B, torch, cfg, batch, slots, dev, stream, graph=args.graph)
    with ClockSampler(local) as clk:
        times, total = run.time(args.steps, args.warmup)
    n_prof = max(1, min(args.steps, 20))
    prof = run.profile(n_prof)
    ms = total / args.steps
    value = cfg.n_tokens / (ms / 1e3)

    # e2e through the C-ABI with host buffers (lora_apply_multi_host)
    e2e = None
    if args.e2e_steps > 0:
        T, ysz = run.T, run.ysz
        xh = {xb: run.xs[xb].cpu().pin_memory() for xb in run.xs}
        xh_list = [xh[cfg.slots[i].xbuf] for i in slots]
        yh = [y.cpu().pin_memory() for y in run.ys]
        adh = batch.adapter_ids.copy()
        exh = batch.expert_ids.copy()
        h2d = adh.nbytes + (exh.nbytes if E > 1 else 0) + sum(v.numel() * 2 for v in xh.values()) + \
            sum(y.numel() * ysz for y in yh)
        d2h = sum(y.numel() * ysz for y in yh)
        B.lora_apply_multi_host(run.s, slots, xh_list, adh, exh if E > 1 else None, yh, run.dt, T, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            B.lora_apply_multi_host(run.s, slots, xh_list, adh, exh if E > 1 else None, yh, run.dt, T, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / args.e2e_steps
        e2e = {"value": cfg.n_tokens / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems, "api": "lora_apply_multi_host (pinned host)"}
        # the paper's protocol: activations up, deltas down, the
        # client adds them -- no base output over PCIe (lora_apply_multi_host_delta)
        dh = [torch.empty_like(y).pin_memory() for y in yh]
        h2d_d = h2d - sum(y.numel() * ysz for y in yh)
        B.lora_apply_multi_host_delta(run.s, slots, xh_list, adh, exh if E > 1 else None, dh, run.dt, T, stream)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            B.lora_apply_multi_host_delta(run.s, slots, xh_list, adh, exh if E > 1 else None, dh, run.dt, T, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1) / args.e2e_steps
        e2e["delta_api"] = {"value": cfg.n_tokens / (dms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d_d),
                            "d2h_bytes_per_step": int(d2h), "ms_per_step": dms,
                            "api": "lora_apply_multi_host_delta (pinned host; x + ids up, deltas down)"}
    run.destroy()

    alg = algorithmic(cfg, batch, slots, int(os.environ.get("LORA_SMALL_SEG_MAX", "8")))
    kern = kernel_table(prof, n_prof, alg)
    # dominant kernel: most device time per step; algorithmic bytes per launch
    dom = max(prof, key=lambda n: kern[n]["ms_per_step"])
    bytes_per_launch = alg.get(dom, 0) * n_prof / kern[dom]["launches"]
    achieved = bytes_per_launch / (kern[dom]["ms_per_launch"] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(cfg.name, {}).get(dom)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic, "kernel": dom,
                "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_src,
                "peak_note": "MEASURED_PEAKS hbm_gbs is a copy (read + write) figure; a read-dominated "
                             "stream can exceed it (tools/bw_probe.cu: 7.35 TB/s bulk-copy read stream)",
                "frac_of_nominal_8TBs": achieved / NOMINAL_HBM_GBS,
                "timing": f"CUDA events on the launching stream, {n_prof} steps right after the timed region "
                          "with the kernels serialised (lora_server_set_concurrent(0))"}
    # kernels per step counted in the profiling pass (same steps, same launches)
    launches = int(round(sum(n for n, _ in prof.values()) / n_prof * args.steps))
    step_gbs = alg["total"] / (ms * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_median": float(np.median(times)),
            "ms_min": float(np.min(times)), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (counter-hash weights/activations, Zipf(1.2) adapter ids, top-2 uniform experts)",
            "config": {"workload": cfg.name, "global_batch": cfg.n_tokens, "rows": batch.n_rows, "slots": len(slots),
                       "rank": cfg.rank, "adapters": cfg.n_adapters, "parallelism": "single GPU",
                       "cuda_graph": bool(run.graph is not None),
                       "l2": f"inputs larger than L2 ({alg['total'] / 1e9:.1f} GB touched per step)"},
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roofline,
            "step_hbm": {"algorithmic_GB": alg["total"] / 1e9, "achieved_GBs": step_gbs,
                         "frac_measured": step_gbs / hbm_peak, "frac_nominal_8TBs": step_gbs / NOMINAL_HBM_GBS,
                         "tflops": alg["flops"] / (ms * 1e-3) / 1e12},
            "kernels": kern,
            "clocks": clk.summary()}
    if args.secondary:
        try:
            line["secondary"] = secondaries(B, torch, dev, stream, hbm_peak, args.secondary_steps, 3)
        except Exception as e:  # a report; the headline stands without it
            line["secondary"] = {"error": str(e)[:300]}
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, batch, slots, args.cpu_seconds)
        except Exception as e:  # the baseline is a report, never the product path
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, cfg, batch, slots):
    """N ranks of the adapter-sharded server (one process per GPU; torchrun).

    The caller's x and y buffers are registered once (lora_shard_register:
    CUDA IPC mappings on every peer); lora_apply_sharded then runs the
    device-side path -- counts exchanged through peer memory, the owner's
    shrink reading x rows from the source's buffer over NVLink, the expand
    epilogue adding the deltas straight into the source's y (push) -- with no
    host synchronisation, so the whole sharded step is captured in a CUDA graph.
    --share-gpu (or more ranks than visible GPUs): every rank on one device
    with the host control plane (gloo), the multi-process check of the same
    path on a single B200."""
    import torch
    import torch.distributed as dist

    from paper_2604_07173_b200 import binding as B
    from paper_2604_07173_b200 import placement as PL

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    share = args.share_gpu or world > ndev
    dev_i = local % ndev
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    k = batch.top_k
    t0, t1 = (cfg.n_tokens * rank) // world, (cfg.n_tokens * (rank + 1)) // world
    r0, r1 = t0 * k, t1 * k
    T = r1 - r0
    E = cfg.slots[slots[0]].n_experts
    dt_code = B.LORA_FP32 if cfg.y_dtype == "fp32" else B.LORA_BF16
    ysz = 4 if cfg.y_dtype == "fp32" else 2
    if world == 1:
        os.environ["LORA_SHARD_LOOPBACK"] = "1"  # every row through the exchange (to itself)

    # popularity-aware placement (R19): replicate the hottest adapters
    # on every rank; auto = the host cost model's choice
    hs, ho, xbf = ([cfg.slots[i].h_in for i in slots], [cfg.slots[i].h_out for i in slots],
                   [cfg.slots[i].xbuf for i in slots])
    ub, rb, xb = PL.slot_bytes(hs, ho, xbf, cfg.rank, ysz, ysz)
    _, _, xpb, dpb = PL.slot_bytes_push(hs, ho, xbf, cfg.rank, ysz, ysz)
    src = PL.sources_of_rows(cfg.n_tokens, k, world)
    # cost model of the path that will run (push when x / y get registered)
    push_kw = {} if args.no_register else {"x_bytes": xpb, "d_bytes": dpb}
    ch = PL.choose_placement(batch.adapter_ids, batch.expert_ids if E > 1 else None, src, world, ub, rb, xb,
                             **push_kw)
    n_rep = ch["n_replicated"] if args.n_replicated < 0 else args.n_replicated
    ep_mode = ch["expert_parallel"] if args.n_replicated < 0 else False
    rep_table = {str(h): round(v * 1e3, 4) for h, v in ch["table"].items()}
    c = B.make_config([sl.h_in for sl in cfg.slots], [sl.h_out for sl in cfg.slots],
                      [sl.n_experts for sl in cfg.slots], cfg.rank, cfg.n_adapters, cfg.scale(), max(T, 1), dev_i,
                      n_replicated=n_rep, expert_parallel=ep_mode)
    if share and world > 1:
        def allgather(data: bytes) -> bytes:
            t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
            out = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return b"".join(o.numpy().tobytes() for o in out)
        s = B.lora_server_create_sharded_host(c, rank, world, allgather)
    else:
        uid = [B.lora_nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        s = B.lora_server_create_sharded(c, rank, world, uid[0])
    B.lora_server_fill_synthetic(s, cfg.seed, stream)

    # device-resident inputs (this rank's rows, global row ids for the generator)
    xs = {}
    for i in slots:
        sl = cfg.slots[i]
        if sl.xbuf not in xs:
            x = torch.empty((max(T, 1), sl.h_in), dtype=torch.int16, device=dev)
            B.lora_synth_fill_rows(x, T, sl.h_in, cfg.seed, li.tag_of(li.KIND_X, sl.xbuf), li.shift_x(), r0, stream)
            xs[sl.xbuf] = x
    x_list = [xs[cfg.slots[i].xbuf] for i in slots]
    ys = []
    for i in slots:
        sl = cfg.slots[i]
        y = torch.empty((max(T, 1), sl.h_out), dtype=torch.int16, device=dev)
        B.lora_synth_fill_rows(y, T, sl.h_out, cfg.seed, li.tag_of(li.KIND_Y0, i), li.shift_y0(), r0, stream)
        if ysz == 4:
            y = ((y.to(torch.int32) << 16).view(torch.float32)).contiguous()
        ys.append(y)
    ad = torch.from_numpy(batch.adapter_ids[r0:r1].copy()).to(dev)
    ex = torch.from_numpy(batch.expert_ids[r0:r1].copy()).to(dev)
    registered = False
    if not args.no_register:
        bufs = list(xs.values()) + ys
        B.lora_shard_register(s, bufs, [b.numel() * b.element_size() for b in bufs], stream)
        registered = True

    def step(st=None):
        B.lora_apply_sharded(s, slots, x_list, ad, ex if E > 1 else None, ys, dt_code, T,
                             stream if st is None else st)

    run_step = step
    graph = None
    if args.graph and registered:
        g_stream = torch.cuda.Stream()
        g_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(g_stream):
            step(g_stream)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=g_stream):
                step(g_stream)
        torch.cuda.current_stream().wait_stream(g_stream)
        run_step = graph.replay
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()
    assert B.lora_server_check(s) == B.LORA_OK, B.lora_last_error(s)
    if world > 1:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev_i) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for kk in range(args.steps):
            run_step()
            ev[kk + 1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    times = [ev[kk].elapsed_time(ev[kk + 1]) for kk in range(args.steps)]
    ms_local = ev[0].elapsed_time(ev[-1]) / args.steps

    def max_over_ranks(v):
        if world == 1:
            return v
        t_ = torch.tensor([v], device="cpu" if share else dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    ms = max_over_ranks(ms_local)
    value = cfg.n_tokens / (ms / 1e3)
    # per-kernel durations on this rank (kernels serialised, eager launches)
    n_prof = 5
    B.lora_server_set_concurrent(s, False)
    B.lora_profile_enable(s, n_prof * 48 + 16)
    for _ in range(n_prof):
        step()
    torch.cuda.synchronize()
    prof = B.lora_profile_read(s)
    B.lora_profile_enable(s, 0)
    B.lora_server_set_concurrent(s, True)
    if world > 1:
        dist.barrier()

    e2e = None
    if args.e2e_steps > 0:
        # this rank's rows from pinned host memory -> lora_apply_sharded -> y back to the host
        xh = {xb_: xs[xb_].cpu().pin_memory() for xb_ in xs}
        yh = [y.cpu().pin_memory() for y in ys]
        adh = ad.cpu().pin_memory()
        exh = ex.cpu().pin_memory()
        h2d = adh.numel() * 4 + (exh.numel() * 4 if E > 1 else 0) + sum(v.numel() * 2 for v in xh.values()) + \
            sum(y.numel() * ysz for y in yh)
        d2h = sum(y.numel() * ysz for y in yh)

        def e2e_step():
            for xb_ in xs:
                xs[xb_].copy_(xh[xb_], non_blocking=True)
            for y, yhh in zip(ys, yh):
                y.copy_(yhh, non_blocking=True)
            ad.copy_(adh, non_blocking=True)
            ex.copy_(exh, non_blocking=True)
            step()
            for y, yhh in zip(ys, yh):
                yhh.copy_(y, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps)
        e2e = {"value": cfg.n_tokens / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems,
               "api": "pinned host -> lora_apply_sharded -> host (per rank; bytes are this rank's)"}
    ok = B.lora_server_check(s)
    B.lora_server_destroy(s)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    hbm_peak, tc_peak, peak_src = load_peaks()
    # the slowest rank's algorithmic HBM bytes (placement model, SURVEY 8d per
    # rank) over the max-over-ranks step time
    rb_ = PL.rank_hbm_bytes(batch.adapter_ids, batch.expert_ids if E > 1 else None, src, world, n_rep, ub, rb,
                            ep=ep_mode)
    achieved = float(rb_.max()) / (ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None, "kernel": "step (slowest rank, all kernels)",
                "algorithmic_bytes_per_launch": float(rb_.max()), "peak_source": peak_src,
                "frac_of_nominal_8TBs": achieved / NOMINAL_HBM_GBS,
                "timing": "CUDA events on the launching stream over the timed region, max over ranks"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_median_rank0": float(np.median(times)),
            "ms_min_rank0": float(np.min(times)), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (counter-hash weights/activations, Zipf(1.2) adapter ids, top-2 uniform experts)",
            "config": {"workload": cfg.name, "global_batch": cfg.n_tokens, "rows": batch.n_rows, "slots": len(slots),
                       "rank": cfg.rank, "adapters": cfg.n_adapters,
                       "parallelism": f"adapter-sharded dp{world}" + (" (ranks share one GPU, host control plane)"
                                                                      if share and world > 1 else ""),
                       "path": "registered buffers: device counts + remote-x shrink + push-add expand"
                               if registered else "unregistered: NCCL send/recv transport",
                       "cuda_graph": graph is not None, "n_replicated": n_rep, "expert_parallel": ep_mode,
                       "placement_model_ms": rep_table,
                       "hybrid_layouts_model_ms": {k_: round(v_ * 1e3, 4) for k_, v_ in PL.hybrid_table(
                           batch.adapter_ids, batch.expert_ids, src, world, ub, rb, xpb, dpb).items()}
                       if E > 1 and world > 1 else None,
                       "l2": "inputs larger than L2"},
            "e2e": e2e,
            "gpu_launches": int(round(sum(n_ for n_, _ in prof.values()) / n_prof * args.steps)),
            "roofline": roofline,
            "kernels_rank0": {k_: {"launches": n_, "ms_per_step": t_ / n_prof} for k_, (n_, t_) in prof.items()},
            "device_errors": int(ok),
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without a torchrun environment: start N ranks
    (one process per GPU) with torch.distributed.run on 127.0.0.1."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    faulthandler.enable()
    # stdout carries exactly one JSON line: keep NCCL's version banner off it
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mixtral_sharded", choices=sorted(li.CONFIGS) + sorted(li.VARIANTS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n-replicated", type=int, default=-1,
                    help="sharded server: adapters [0, h) stored on every rank; -1 = cost-model choice")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch every step eagerly (default: one step captured in a CUDA graph, replayed)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the sharded server even at N=1 with every row sent through the exchange "
                         "(loopback; exercises the N>1 code path)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="N>1: every rank on one GPU (host control plane over gloo)")
    ap.add_argument("--no-register", action="store_true",
                    help="sharded: do not register x / y (NCCL send/recv transport, one host sync per step)")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false",
                    help="skip configs 3 / 2 / 4 and the E10 / E13 sweeps after the headline")
    ap.add_argument("--secondary-steps", type=int, default=20)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    cfg = li.CONFIGS[args.workload] if args.workload in li.CONFIGS else li.VARIANTS[args.workload]
    batch = li.make_batch(cfg)
    slots = list(range(len(cfg.slots)))
    if args.impl == "reference":
        return run_reference(args, cfg, batch, slots)
    return run_ours(args, cfg, batch, slots)


if __name__ == "__main__":
    sys.exit(main())
