#!/usr/bin/env python
"""Benchmark: batched AGFT tuner replay, tuner-steps/s on N B200s (BASELINE.json metric).

Workload (one "step" = one pass of the whole hot path, SURVEY §8 rows a0–a11):
BASELINE configs[3] = C4 — 65,536 tuners per GPU (16 α0 × 16 pruning settings × 256
traces, diurnal + burst load), the full 107-arm grid, d = 7, 24 h = 108,000 decision
windows.  Per step: reset tuners → [trace records (K1) → replay (K2)] × 24 chunks →
stats (→ NCCL all-gather of stats and a 16×u64 counter all-reduce when N > 1).  Strong
scaling: the 65,536 tuners and their 256 traces are split over the N ranks
(65,536/N tuners per GPU, whole traces per rank, no input exchange).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

``--impl reference`` times the CPU oracle (the paper has no code; oracle/ is this
tier's reference arm) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tuner-steps/sec (device-timed) at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "tuner-steps/s"
CHUNK = 4500                     # decision windows per replay launch (1 h of trace)
FP64_UNITS_PER_SM = 64           # FP64 FMA lanes per SM (B200)
N_SM = 148
STATS_DTYPE_BYTES = 128


def src_sha() -> str:
    """Hash of the CUDA sources and the ABI header: ties an ncu capture to the build it measured."""
    import hashlib
    h = hashlib.sha256()
    for d in (os.path.join(ROOT, "paper_2508_01744_b200", "csrc"), os.path.join(ROOT, "include")):
        for name in sorted(os.listdir(d)):
            if name.endswith((".cu", ".cuh", ".h")):
                with open(os.path.join(d, name), "rb") as f:
                    h.update(name.encode() + b"\0" + f.read())
    return h.hexdigest()[:16]


def profile_traffic(workload_key: str):
    """ncu DRAM read + write bytes per launch of each replay class, from the capture of one bench step
    of THIS build and workload (tools/ncu_traffic.py → profiles/*_traffic.json, matched on the source
    hash and the workload key), or None when no capture of this build exists."""
    import glob
    sha = src_sha()
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")), reverse=True):
        try:
            with open(path) as f:
                tr = json.load(f)
        except (OSError, ValueError):
            continue
        if tr.get("src_sha") == sha and tr.get("workload_key") == workload_key:
            tr["source"] = os.path.relpath(path, ROOT)
            return tr
    return None


def latency_roofline():
    """Per-class latency ceilings (resident tuners ÷ chain latency per window) measured for THIS build by
    tools/latency_roofline.py (profiles/*latency_roofline.json, matched on the source hash), or None."""
    import glob
    sha = src_sha()
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*latency_roofline.json")), reverse=True):
        try:
            with open(path) as f:
                lr = json.load(f)
        except (OSError, ValueError):
            continue
        if lr.get("src_sha") == sha:
            lr["source"] = os.path.relpath(path, ROOT)
            return lr
    return None


def measured_fp64_peak():
    """FP64 DFMA TFLOP/s measured on a B200 of this pool by tools/fp64_peak.cu (profiles/*fp64_peak.json)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*fp64_peak.json")), reverse=True):
        try:
            with open(path) as f:
                return float(json.load(f)["fp64_dfma_tflops"]), os.path.relpath(path, ROOT)
        except (OSError, ValueError, KeyError):
            continue
    return None, None


def flops_per_step(d: int, k_act_sum: float, steps: float) -> float:
    """Algorithmic FP64 flops: per active arm d²+3d+3 (Eq. 1 score) + 5
    (pruning bookkeeping); per step 3d²+8d+4 (Sherman–Morrison + RLS update) + 50
    (response, reward, Welford, stats)."""
    return k_act_sum * (d * d + 3 * d + 3 + 5) + steps * (3 * d * d + 8 * d + 4 + 50)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def parity_sample(cfg: dict, n: int, k: int = 256) -> list:
    """The tuners the cpu_baseline leg replays through the oracle: for the α × pruning sweep, every
    4th hyper-parameter point of four traces spread over the shard (diurnal and burst patterns),
    else the first k tuners."""
    if cfg.get("sweep") == "hyper256" and n >= 1024 and n % 256 == 0:
        R = n // 256
        traces = sorted({0, R // 3, (2 * R) // 3, R - 1}) if R >= 4 else list(range(R))
        per = k // len(traces)
        step = max(1, 256 // per)
        return [r * 256 + h for r in traces for h in range(0, 256, step)][:k]
    return list(range(min(k, n)))


def run_cpu_baseline(cfg: dict, ids: list, T: int) -> dict:
    """The oracle as it stands on this host's cores, on a bounded sample of the workload."""
    import oracle
    from agft_inputs import tuner_params
    n_tuners = len(ids)
    params = tuner_params(cfg, list(ids))
    cores = os.cpu_count() or 1
    t = time.perf_counter()
    ost = oracle.run_batch(cfg, params, T, threads=cores)
    dt = time.perf_counter() - t
    n1 = min(4, n_tuners)                              # the 1-thread rate beside it
    t1 = time.perf_counter()
    oracle.run_batch(cfg, tuner_params(cfg, list(ids[:n1])), T, threads=1)
    dt1 = time.perf_counter() - t1
    return {"value": n_tuners * T / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "one_thread_value": n1 * T / dt1, "one_thread_sample": f"{n1} tuners × {T} steps, 1 thread",
            "sample": f"{cfg.get('name', 'C4')}: {n_tuners} tuners (traces "
                      f"{sorted({int(t) for t in params['trace_id']})}, "
                      f"{len(set(int(i) % 256 for i in ids))} hyper-parameter points each) × {T} steps, "
                      f"free-running, {dt:.1f} s on {cores} threads"}, ost


PARITY_EXACT = ("steps", "n_active", "sum_active", "n_pruned_extreme", "n_pruned_hist", "n_pruned_cascade",
                "sum_energy", "sum_tpot", "sum_ttft", "sum_edp", "sum_reward", "base_energy", "base_edp")


def arm_state_errors(cfg, params, tb, T, sample) -> dict:
    """the largest relative error of A⁻¹ and θ (Sherman–Morrison on the GPU against
    Gauss–Jordan / solve in the oracle, ENV.md §4.3) over a few tuners of the timed run, and whether
    their counters and b match exactly; the oracle runs each tuner's full day single-threaded."""
    import oracle
    worst_a = worst_t = 0.0
    exact = 0
    for i in sample:
        tu = oracle.make_tuner(int(params["trace_id"][i]), params["alpha0"][i], params["ext_reward_threshold"][i],
                               params["hist_k"][i])
        _, oa, _ = oracle.run_tuner(cfg, tu, T=T)
        g = tb.export_arms(i)
        for name, key in (("Ainv", "a"), ("theta", "t")):
            go, oo = np.asarray(g[name]), np.asarray(oa[name])
            err = float(np.max(np.abs(go - oo) / np.maximum(np.max(np.abs(oo), axis=tuple(range(1, oo.ndim)),
                                                                    keepdims=True), 1e-300)))
            if key == "a":
                worst_a = max(worst_a, err)
            else:
                worst_t = max(worst_t, err)
        exact += int(all(np.array_equal(np.asarray(g[f]).astype(np.float64), np.asarray(oa[f]).astype(np.float64))
                         for f in ("n", "b", "rbar", "ebar", "active")))
    return {"arm_state_tuners": list(sample), "ainv_max_rel_err": worst_a, "theta_max_rel_err": worst_t,
            "arm_counters_b_exact": exact, "arm_state_tolerance": 1e-9}


def parity_summary(gst, ost, ids=None) -> dict:
    """The timed run's own statistics for the tuners the cpu_baseline leg ran through the oracle
    (same config, same windows): trajectory-hash matches and, for those, exact equality of every
    counter and fp64 sum (ENV.md §0).  A free-running oracle may leave the GPU's path at a near-tie
    (ENV.md §4.5); the GPU's near-tie count is reported beside it."""
    ids = list(range(min(len(ost), len(gst)))) if ids is None else list(ids)
    n = len(ids)
    match = [j for j, i in enumerate(ids) if int(gst["traj_hash"][i]) == ost[j]["traj_hash"]]
    exact = [j for j in match if all(gst[f][ids[j]] == ost[j][f] for f in PARITY_EXACT)]
    return {"tuners": n, "traj_hash_match": len(match), "stats_exact_given_traj": len(exact),
            "near_tie_steps_gpu": int(gst["near_tie_steps"][ids].astype(np.int64).sum()),
            "fields": list(PARITY_EXACT),
            "oracle": "free-running fp64 C oracle of the cpu_baseline leg, same config and windows"}


def workload_key(args, cfg, n, R, T, chunk) -> str:
    return (f"{args.config}:n={n}:R={R}:T={T}:ph={int(bool(cfg.get('ph_enable')))}:rf={int(bool(cfg.get('rf_enable')))}"
            f":cl={int(cfg.get('cl_enable', 0))}:pol={args.policy}:chunk={chunk}")


def class_roofline(d, prof, prof_conc, steps, replay_ms, serial_replay_ms, st, n, T, R, traffic) -> dict:
    """SURVEY §8(d) roofline per replay class (agft_profile_*: tuner-steps and Σ K_act each class's
    kernels processed, and CUDA-event times of its launches).  ``prof`` is one C4 day with every class
    kernel alone on the stream (per-kernel durations); ``prof_conc`` the timed region itself, where
    the classes of a sub-chunk run concurrently on their own streams (a class's event span includes
    its wait for SMs held by the others).  Algorithmic flops ÷ the kernel's own time,
    against the FP64 peak; the dominant kernel is the class with the most kernel time."""
    pk = peaks()
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    peak_fp64 = N_SM * FP64_UNITS_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    meas, meas_src = measured_fp64_peak()
    lat = latency_roofline()
    classes = {}
    for name, c in prof.items():
        if not c["launches"]:
            continue
        e = {"launches": c["launches"], "kernel_ms": round(c["kernel_ms"], 3),
             "ms_per_launch": round(c["kernel_ms"] / c["launches"], 4)}
        if c["tuner_steps"]:
            fl = flops_per_step(d, float(c["active_arm_steps"]), float(c["tuner_steps"]))
            ach = fl / (c["kernel_ms"] / 1e3) / 1e12
            e.update({"share_of_serial_step": round(c["kernel_ms"] / serial_replay_ms, 4),
                      "concurrent_span_ms_per_step": round(prof_conc[name]["kernel_ms"] / steps, 3),
                      "tuner_steps": c["tuner_steps"], "mean_active_arms": round(c["active_arm_steps"] / c["tuner_steps"], 3),
                      "tuner_steps_per_s": round(c["tuner_steps"] / (c["kernel_ms"] / 1e3), 1),
                      "achieved_tflops": round(ach, 4), "frac": round(ach / peak_fp64, 5)})
        if lat and name in lat.get("classes", {}) and "tuner_steps_per_s" in e:
            ceil = lat["classes"][name]["latency_ceiling_tuner_steps_per_s"]
            e["latency_ceiling_tuner_steps_per_s"] = ceil
            e["frac_of_latency_ceiling"] = round(e["tuner_steps_per_s"] / ceil, 4)
        if traffic and name in traffic.get("classes", {}):
            tc = traffic["classes"][name]
            e["traffic_per_launch"] = tc["dram_bytes"] / max(1, tc["launches"])
        classes[name] = e
    replay = {k: v for k, v in classes.items() if "tuner_steps" in v}
    top = max(replay, key=lambda k: replay[k]["kernel_ms"]) if replay else None
    sum_active = float(np.sum(st["sum_active"], dtype=np.float64))
    step_flops = flops_per_step(d, sum_active, float(n) * T) * steps
    out = {"bound": "alu", "kernel": top, "unit": "TFLOP/s",
           "peak": round(peak_fp64, 2),
           "peak_source": "derived: 148 SM × 64 FP64 FMA/clk × 2 × sm_max_mhz (DESIGN.md §5)",
           "peak_measured": meas, "peak_measured_source": meas_src}
    if top:
        t = replay[top]
        out.update({"achieved": t["achieved_tflops"], "frac": t["frac"],
                    "frac_of_measured_peak": round(t["achieved_tflops"] / meas, 5) if meas else None,
                    "traffic": t.get("traffic_per_launch")})
    out.update({"attribution": "one extra C4 day with each class kernel alone on the stream (agft_profile_start(h, 1)); "
                               f"serialised replay {serial_replay_ms:.1f} ms vs {replay_ms / steps:.1f} ms concurrent",
                "whole_replay": {"achieved_tflops": round(step_flops / (replay_ms / 1e3) / 1e12, 4),
                                 "frac": round(step_flops / (replay_ms / 1e3) / 1e12 / peak_fp64, 5),
                                 "replay_ms": round(replay_ms, 3), "mean_active_arms": round(sum_active / (float(n) * T), 3)},
                "classes": classes,
                "latency_roofline": ({"source": lat["source"], "bound": "latency: resident tuners ÷ chain latency per "
                                      "window, per class at its full K (tools/latency_roofline.py)"}
                                     if lat else None),
                "traffic_source": traffic.get("source") if traffic else None,
                "traffic_total_bytes_per_step": traffic.get("total_dram_bytes") if traffic else None,
                # records once (128 B per window and trace) + the stats
                "algorithmic_hbm_bytes_per_step": 128 * T * R + STATS_DTYPE_BYTES * n})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--T", type=int, default=None, help="override decision windows (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--closed", action="store_true",
                    help="ENV-C closed-loop environment (ENV.md §6; raw rows alongside the records)")
    ap.add_argument("--des", action="store_true",
                    help="ENV-S: every tuner on its own discrete-event continuous-batching server (ENV.md §7)")
    ap.add_argument("--refine", action="store_true",
                    help="enable mixed maturity-based refinement (ENV.md §4.11; class schedule + refinement passes)")
    ap.add_argument("--chunk", type=int, default=CHUNK, help="windows per agft_replay call (records buffer)")
    ap.add_argument("--phase", action="store_true",
                    help="enable the Page-Hinkley exploitation phase (ENV.md §4.10; not the §8(a) headline)")
    ap.add_argument("--policy", type=int, default=int(os.environ.get("AGFT_POLICY", "0")),
                    help="0 auto (SOLO/SEG/WIDE), 1 wide only, 2 SOLO/MSEG/WIDE")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="strong: split the config's tuners over the ranks (default for C4, C5); weak: every rank "
                         "runs the full config (default for C1-C3)")
    ap.add_argument("--backend", default="nccl", help="process-group backend for N > 1 (nccl; gloo for tests)")
    ap.add_argument("--workload", default="replay", choices=["replay", "sweep", "live"],
                    help="replay: the tuner hot path (north-star metric); sweep: ENV.md §5 offline sweep; "
                         "live: agft_select/agft_observe decision latency")
    ap.add_argument("--tuners", type=int, default=1024, help="live workload: tuners per GPU")
    args = ap.parse_args()
    if args.scaling is None:                 # C4 and C5 split their tuners over the ranks
        args.scaling = "strong" if args.config in ("C4", "C5") else "weak"

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from agft_inputs import named_config, tuner_params
    cfg = named_config(args.config)
    if args.T:
        cfg["T"] = args.T
    if args.phase:
        cfg["ph_enable"] = 1          # ENV.md §4.10 exploitation phase
    if args.refine:
        cfg["rf_enable"] = 1          # ENV.md §4.11 refinement (NEXT row 1)
    if args.closed:
        cfg["cl_enable"] = 1          # ENV.md §6 closed loop (NEXT row 3)
    if args.des:
        cfg["cl_enable"] = 2          # ENV.md §7 ENV-S discrete-event servers (NEXT row 3)
    T = cfg["T"]

    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)
    if args.workload == "sweep":
        return sweep_bench(args, cfg, rank, world, local)
    if args.workload == "live":
        return live_bench(args, cfg, rank, world, local)

    import numpy as np
    import torch
    import paper_2508_01744_b200 as pkg
    from paper_2508_01744_b200 import TunerBatch, STATS_DTYPE

    from paper_2508_01744_b200 import shard
    local = local % max(1, torch.cuda.device_count())   # >1 rank per GPU only for gloo smoke tests
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.backend)

    sh = shard.plan(cfg, world, rank, args.scaling)
    n, R = sh.n_tuners, sh.n_traces
    cfg = dict(cfg, n_tuners=n, n_traces=R)
    params = sh.params                                # local trace ids 0..R-1
    tb = TunerBatch(cfg, params, device=f"cuda:{local}", trace_base=sh.trace_base, policy=args.policy)
    stream = torch.cuda.current_stream()
    chunk = min(args.chunk, T)
    records = tb.new_records(chunk)
    raw = (torch.empty((R, chunk, pkg.ROW_WORDS), dtype=torch.int32, device=f"cuda:{local}")
           if cfg.get("cl_enable") else None)
    stats_out = tb.stats_tensor()
    coll_dev = stats_out.device if args.backend == "nccl" else torch.device("cpu")
    gathered = (torch.empty(world * stats_out.numel(), dtype=torch.uint8, device=coll_dev)
                if world > 1 else None)
    n_chunks = (T + chunk - 1) // chunk
    ev_replay = []

    def one_step(timed: bool):
        tb.reset()
        t = 0
        while t < T:
            m = min(chunk, T - t)
            pkg.agft_trace_generate(tb.h, t, m, records, raw)
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tb.replay(records, t, m, raw=raw)
                e1.record(stream)
                ev_replay.append((e0, e1))
            else:
                tb.replay(records, t, m, raw=raw)
            t += m
        pkg.agft_stats(tb.h, stats_out)
        if world > 1:
            dist.all_gather_into_tensor(gathered, stats_out.to(coll_dev))

    for _ in range(args.warmup):
        one_step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    from paper_2508_01744_b200 import _abi
    launches0 = _abi.lib().agft_kernel_launches()
    pkg.agft_profile_start(tb.h)
    start.record(stream)
    for _ in range(args.steps):
        one_step(True)
    end.record(stream)
    launches = int(_abi.lib().agft_kernel_launches() - launches0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    prof_conc = pkg.agft_profile_read(tb.h)
    ms = start.elapsed_time(end)
    replay_ms = sum(a.elapsed_time(b) for a, b in ev_replay)
    # per-kernel attribution: one more step, untimed for the headline, with every class
    # kernel alone on the stream so that each CUDA-event pair times exactly one kernel
    pkg.agft_profile_start(tb.h, serialize=True)
    ev_replay.clear()
    one_step(True)
    torch.cuda.synchronize()
    prof = pkg.agft_profile_read(tb.h)
    serial_replay_ms = sum(a.elapsed_time(b) for a, b in ev_replay)
    if world > 1:
        t_ = torch.tensor([ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_.item())

    st = stats_out.cpu().numpy().view(STATS_DTYPE)
    steps_ok = bool(np.all(st["steps"] == T)) and bool(np.all(st["flags"] == 0))
    units = float(n) * T * world * args.steps
    value = units / (ms / 1e3)
    # one 16×u64 counter all-reduce (steps, flags, near-ties, invariant violations)
    counters = shard.reduce_counters(shard.counter_vector(st, T), coll_dev) if world > 1 else \
        dict(zip(shard.COUNTER_NAMES, shard.counter_vector(st, T)))

    wkey = workload_key(args, cfg, n, R, T, chunk)
    roofline = class_roofline(cfg["d"], prof, prof_conc, args.steps, replay_ms, serial_replay_ms, st, n, T, R,
                              profile_traffic(wkey))
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config}: {n} tuners/GPU × {cfg['n_arms']} arms × d={cfg['d']} × "
                                  f"{T} windows ({R} traces/GPU{', α×pruning sweep' if cfg.get('sweep') == 'hyper256' else ''}, "
                                  f"{['fluctuating', 'diurnal', 'burst', 'fluct/diurnal/burst', 'diurnal+burst'][cfg['pattern_mode']]})",
                      "tuners_per_gpu": n, "T": T, "arms": cfg["n_arms"], "d": cfg["d"],
                      "phase_switch": bool(cfg.get("ph_enable", 0)),
                      "refinement": bool(cfg.get("rf_enable", 0)),
                      "closed_loop": ["open", "ENV-C backlog", "ENV-S discrete-event servers"][cfg.get("cl_enable", 0)],
                      "traces_per_gpu": R, "chunk": chunk,
                      "l2": f"inputs larger than L2: tuner state {tb.workspace.numel() / 2**30:.2f} GiB/GPU",
                      "parallelism": f"tuner shards dp{world}"},
           "roofline": roofline, "clocks": clk,
           "gpu_launches": launches, "all_steps_complete": steps_ok, "counters": counters}

    if not args.no_e2e:
        out["e2e"] = e2e_leg(cfg, params, sh.trace_base, world, local, chunk, n, T, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ids = parity_sample(cfg, n)
        out["cpu_baseline"], ost = run_cpu_baseline(cfg, ids, T)
        out["parity"] = parity_summary(st, ost, ids)
        out["parity"].update(arm_state_errors(cfg, params, tb, T, [ids[j] for j in (0, 63, 128, 255) if j < len(ids)]))
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


SWEEP_FLOPS = 21   # ENV.md §3.3 without TTFT (13 mul/add, 1 sub, 1 div) + 4 accumulations (§5)


def sweep_bench(args, cfg, rank, world, local):
    """ENV.md §5 offline sweep over the whole day (every trace × every arm × every window):
    one step = trace records (K1) + sweep (K4) for all chunks + Table-6 arms (K5a)."""
    import torch
    from paper_2508_01744_b200 import TunerBatch
    from paper_2508_01744_b200 import shard
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(args.backend, device_id=torch.device("cuda", local)) if args.backend == "nccl" \
            else dist.init_process_group(args.backend)
    sh = shard.plan(cfg, world, rank, args.scaling)
    R, T, K = sh.n_traces, cfg["T"], cfg["n_arms"]
    c = dict(cfg, n_tuners=sh.n_tuners, n_traces=R)
    tb = TunerBatch(c, sh.params, device=f"cuda:{local}", trace_base=sh.trace_base)
    stream = torch.cuda.current_stream()
    chunk = min(CHUNK, T)
    records = tb.new_records(chunk)
    ev = []

    def one(timed):
        sums = tb.new_sweep()
        tb.reset()
        t = 0
        while t < T:
            m = min(chunk, T - t)
            tb.generate(t, m, records)
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tb.sweep(records, t, m, sums)
                e1.record(stream)
                ev.append((e0, e1, m))
            else:
                tb.sweep(records, t, m, sums)
            t += m
        tb.regret(sums)
        return sums

    for _ in range(args.warmup):
        one(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from paper_2508_01744_b200 import _abi
    launches0 = _abi.lib().agft_kernel_launches()
    start.record(stream)
    for _ in range(args.steps):
        sums = one(True)
    end.record(stream)
    launches = int(_abi.lib().agft_kernel_launches() - launches0)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = start.elapsed_time(end)
    if world > 1:
        import torch.distributed as dist
        t_ = torch.tensor([ms], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_.item())
    k_ms = sum(a.elapsed_time(b) for a, b, _ in ev)
    evals = float(R) * K * T
    achieved = evals * SWEEP_FLOPS * args.steps / (k_ms / 1e3) / 1e12
    pk = peaks()
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    peak_fp64 = N_SM * FP64_UNITS_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    h = sums.host()
    out = {"metric": "offline-sweep window-arm evaluations/s (ENV.md §5)", "value": round(evals * world * args.steps / (ms / 1e3), 1),
           "unit": "window-arm evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": args.scaling,
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config} sweep: {R} traces × {K} arms × {T} windows",
                      "traces_per_gpu": R, "arms": K, "T": T, "chunk": chunk},
           "roofline": {"bound": "alu", "achieved": round(achieved, 4), "peak": round(peak_fp64, 2),
                        "unit": "TFLOP/s", "frac": round(achieved / peak_fp64, 5), "traffic": None,
                        "kernel": "sweep_kernel", "kernel_share": round(k_ms / ms, 4),
                        "flops_per_eval": SWEEP_FLOPS,
                        "peak_source": "derived: 148 SM × 64 FP64 FMA/clk × 2 × sm_max_mhz (DESIGN.md §5)"},
           "clocks": clk, "gpu_launches": launches,
           "check": {"windows_counted": int(h["NP"].sum()) == R * T,
                     "oracle_le_fixed": bool(np.all(h["O"][:, 0][:, None] <= h["S"][:, :, 2]))}}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def live_bench(args, cfg, rank, world, local):
    """Live two-phase step (agft_select → measured response → agft_observe):
    one step = T windows for N tuners.  Device leg: snapshot rows and responses already in HBM
    (the response of window t is a seeded measurement table, independent of the arm chosen);
    e2e leg: every window copies the rows host→device, the chosen arms device→host (the
    controller must set the clocks) and the measured responses host→device — the real loop."""
    import torch
    from agft_inputs import live_inputs, tuner_params
    from paper_2508_01744_b200 import TunerBatch, _abi
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(args.backend, device_id=torch.device("cuda", local)) if args.backend == "nccl" \
            else dist.init_process_group(args.backend)
    n = args.tuners
    T = min(cfg["T"], args.T or 2000)
    c = dict(cfg, n_tuners=n, n_traces=n, sweep="none")
    params = tuner_params(c)
    rows, resp = live_inputs(dict(c, n_arms=1), n, T, seed=17 + rank)      # one measurement per window
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    rows_h = torch.from_numpy(np.ascontiguousarray(rows.transpose(1, 0, 2)).view(np.int32)).pin_memory()
    resp_h = torch.from_numpy(np.ascontiguousarray(resp[:, :, 0, :].transpose(1, 0, 2))).pin_memory()
    rows_d, resp_d = rows_h.to(dev), resp_h.to(dev)
    tb = TunerBatch(c, params, device=dev)
    stream = torch.cuda.current_stream()
    chosen = torch.empty((T, n), dtype=torch.int32, device=dev)

    def one(e2e=False):
        tb.reset()
        if not e2e:
            for t in range(T):
                tb.select(rows_d[t], chosen[t])
                tb.observe(resp_d[t])
            return None
        r_buf = torch.empty((n, 12), dtype=torch.int32, device=dev)
        m_buf = torch.empty((n, 3), dtype=torch.float64, device=dev)
        ch_h = torch.empty(n, dtype=torch.int32).pin_memory()
        for t in range(T):
            r_buf.copy_(rows_h[t], non_blocking=True)
            tb.select(r_buf, chosen[t])
            ch_h.copy_(chosen[t], non_blocking=True)
            torch.cuda.current_stream().synchronize()      # the controller applies the clocks here
            m_buf.copy_(resp_h[t], non_blocking=True)
            tb.observe(m_buf)
        return None

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    st0 = tb.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _abi.lib().agft_kernel_launches()
    e0.record(stream)
    for _ in range(args.steps):
        one()
    e1.record(stream)
    launches = int(_abi.lib().agft_kernel_launches() - launches0)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    st = tb.stats()
    k_act = float(st["sum_active"].astype(np.float64).sum())          # last step's Σ K_act
    # e2e: host rows in, chosen arms out, host measurements in, every window
    one(e2e=True)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        one(e2e=True)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = f0.elapsed_time(f1)
    if world > 1:
        import torch.distributed as dist
        t_ = torch.tensor([ms, ms_e2e], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t_[0]), float(t_[1])
    decisions = float(n) * T * args.steps
    pk = peaks()
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    peak_fp64 = N_SM * FP64_UNITS_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    d = c["d"]
    P = d * (d + 1) // 2
    # algorithmic HBM bytes (live): select reads the row (48), mask (16), stats (128),
    # the scored arms' A⁻¹, θ, n ((P+d)·8 + 4 each) and writes the pending record (64) and k* (4);
    # observe reads the measurement (24) and pending record (64), reads and writes the chosen arm's
    # A⁻¹, θ, b and n, r̄, ē (2·((P+2d)·8 + 20)), reads n, r̄, ē of the active arms (20 each), and
    # reads and writes the EDP window (2·1 KiB), the stats (2·128) and the mask (16)
    per_dec = (48 + 16 + 128 + 64 + 4) + (24 + 64 + 2 * ((P + 2 * d) * 8 + 20) + 2 * 1024 + 2 * 128 + 16)
    per_arm = (P + d) * 8 + 4 + 20
    alg_bytes = (float(n) * T * per_dec + k_act * per_arm) * args.steps
    achieved = alg_bytes / (ms / 1e3) / 1e9
    peak_hbm = float(pk.get("hbm_gbs", 7700.0))
    out = {"metric": "live decisions/s (agft_select + agft_observe, device-timed)",
           "value": round(decisions * world / (ms / 1e3), 1), "unit": "tuner-decisions/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (agft_inputs.live_inputs snapshots + measurement table)",
           "config": {"workload": f"live: {n} tuners × {c['n_arms']} arms × d={c['d']} × {T} windows",
                      "tuners_per_gpu": n, "T": T, "us_per_window": round(ms * 1e3 / (T * args.steps), 2),
                      "mean_active_arms": round(k_act / (float(n) * T), 3),
                      "l2": "tuner state 80 KB/tuner: above L2 from ~1,500 tuners"},
           "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": round(peak_hbm, 1),
                        "unit": "GB/s", "frac": round(achieved / peak_hbm, 5), "traffic": None,
                        "kernel": "replay_kernel<MODE 1|2> (the only launches of the step, besides one reset)",
                        "algorithmic_bytes_per_decision": round(per_dec + per_arm * k_act / (float(n) * T), 1),
                        "fp64_frac": round(flops_per_step(d, k_act, float(n) * T) * args.steps / (ms / 1e3) / 1e12
                                           / peak_fp64, 6),
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
           "clocks": clk, "gpu_launches": launches,
           "e2e": {"value": round(decisions * world / (ms_e2e / 1e3), 1), "unit": "tuner-decisions/s",
                   "h2d_bytes_per_step": n * T * (48 + 24), "d2h_bytes_per_step": n * T * 4,
                   "us_per_window": round(ms_e2e * 1e3 / (T * args.steps), 2),
                   "api": "agft_select/agft_observe with host rows/measurements in and chosen arms out each window"}}
    if rank == 0:
        print(json.dumps(out), flush=True)
    tb.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def e2e_leg(cfg, params, trace_base, world, local, chunk, n, T, args) -> dict:
    """Same metric through agft_run with HOST params/stats: H2D of the per-tuner params and
    D2H of the per-tuner stats are inside the timed region, every step."""
    import numpy as np
    import torch
    import paper_2508_01744_b200 as pkg
    from paper_2508_01744_b200 import make_config, make_params, STATS_DTYPE
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    cfg_c = make_config(cfg, n_tuners=n, n_traces=cfg["n_traces"], trace_base=trace_base,
                        policy=args.policy)
    ws = torch.empty(pkg.agft_workspace_bytes(cfg_c), dtype=torch.uint8, device=dev)
    per = pkg.RECORD_BYTES + (pkg.ROW_WORDS * 4 if cfg.get("cl_enable") else 0)   # + raw rows (ENV.md §6)
    scratch = torch.empty(cfg["n_traces"] * chunk * per, dtype=torch.uint8, device=dev)
    hp = torch.from_numpy(make_params(params).view(np.uint8)).pin_memory()
    dp = torch.empty_like(hp, device=dev)
    ds = torch.empty(n * STATS_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    hs = torch.empty(n * STATS_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    pkg.agft_run(cfg_c, hp, dp, T, chunk, ws, scratch, ds, hs)          # warm-up
    reps = max(1, min(args.steps, 2))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t = time.perf_counter()
    for _ in range(reps):
        pkg.agft_run(cfg_c, hp, dp, T, chunk, ws, scratch, ds, hs)
    dt = time.perf_counter() - t
    if world > 1:
        import torch.distributed as dist
        t_ = torch.tensor([dt], dtype=torch.float64, device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        dt = float(t_.item())
    return {"value": round(n * T * world * reps / dt, 1), "unit": UNIT, "h2d_bytes_per_step": hp.numel(),
            "d2h_bytes_per_step": hs.numel(), "api": "agft_run (host params in, host stats out)",
            "steps": reps}


def reference_arm(args, cfg, rank, world):
    """The oracle (this tier's reference arm) on the box's host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle
    from agft_inputs import tuner_params
    T = cfg["T"]
    n_sample = 64
    params = tuner_params(cfg, list(range(n_sample)))
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.run_batch(cfg, params, min(T, 2000), threads=cores)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.run_batch(cfg, params, T, threads=cores)
    dt = time.perf_counter() - t
    value = n_sample * T * args.steps / dt
    sample = f"C4 tuners 0..{n_sample - 1} × {T} windows per step, free-running"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config} (bounded sample)", "sample": sample},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
        flush=True)


if __name__ == "__main__":
    main()
