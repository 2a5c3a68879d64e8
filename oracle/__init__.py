"""CPU oracle of the AGFT hot path — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over ``oracle/agft_oracle.c`` (plain fp64 C written from the
paper and ENV.md). Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the product
package ``paper_2508_01744_b200`` never does, and the two share no code.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "agft_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11",
          "-Wall", "-Wextra"]


def build(force: bool = False) -> str:
    """Compile the oracle with the ENV.md §0 floating-point flags."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "agft_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB, SRC, "-lm", "-lpthread"])
    return LIB


u32, u64, f64 = C.c_uint32, C.c_uint64, C.c_double


class OrcConfig(C.Structure):
    _fields_ = [
        ("f_min_mhz", u32), ("f_step_mhz", u32), ("n_arms", u32), ("f_max_hw_mhz", u32),
        ("d", u32), ("median_window", u32), ("prune_enable", u32),
        ("ext_round_limit", u32), ("ext_min_samples", u32), ("hist_min_round", u32),
        ("hist_min_samples", u32), ("pattern_mode", u32),
        ("seg_steps", u32), ("steps_per_hour", u32), ("burst_steps", u32), ("burst_p32", u32),
        ("cap", u32), ("kv_total", u32),
        ("ctx_lo", u32 * 5), ("ctx_hi", u32 * 5), ("gen_lo", u32 * 5), ("gen_hi", u32 * 5),
        ("weight", u32 * 5), ("pad0", u32),
        ("seed", u64),
        ("norm_lo", f64 * 7), ("norm_hi", f64 * 7),
        ("tau", f64), ("clip_lo", f64), ("clip_hi", f64), ("cascade_fraction", f64), ("tie_rel", f64),
        ("W", f64), ("p_idle", f64), ("k_lin", f64), ("k_cube", f64), ("u_floor", f64),
        ("u_max", f64), ("c_p", f64), ("c_d", f64), ("beta", f64), ("sigma_e", f64), ("sigma_t", f64),
        ("lambda0", f64), ("burst_mult", f64), ("t_iter0", f64), ("t_iter1", f64), ("e2e0", f64),
        ("tau_ref", f64),
        ("conc_mult", f64 * 5), ("hit_rate", f64 * 5), ("knot", f64 * 24),
        ("ph_enable", u32), ("ph_window", u32), ("ph_delta", f64), ("ph_lambda", f64),
        ("rf_enable", u32), ("rf_period", u32), ("rf_mature", u32), ("rf_min_samples", u32),
        ("rf_half_mhz", u32), ("rf_step_mhz", u32),
        ("cl_enable", u32), ("cl_q_max", u32),
    ]


class OrcTuner(C.Structure):
    _fields_ = [("trace_id", u32), ("pad", u32), ("alpha0", f64),
                ("ext_reward_threshold", f64), ("hist_k", f64)]


class OrcStats(C.Structure):
    _fields_ = [("traj_hash", u64), ("sum_active", u64),
                ("steps", u32), ("last_arm", u32), ("n_active", u32), ("n_pruned_extreme", u32),
                ("n_pruned_hist", u32), ("n_pruned_cascade", u32), ("near_tie_steps", u32),
                ("follow_violations", u32),
                ("sum_energy", f64), ("sum_tpot", f64), ("sum_ttft", f64), ("sum_edp", f64),
                ("sum_reward", f64), ("base_energy", f64), ("base_edp", f64), ("max_viol_rel", f64),
                ("exploit_steps", u32), ("ph_alarms", u32), ("first_exploit_t", u32), ("phase", u32),
                ("n_refine", u32), ("last_anchor", u32)]


MAXK, MAXD = 128, 7


class OrcStepRec(C.Structure):
    _fields_ = [("x", f64 * 7), ("g", f64), ("invIm", f64), ("invAm", f64), ("wIm", f64),
                ("nT", f64), ("nE", f64), ("baseE", f64), ("baseEDP", f64), ("I", u32), ("P", u32)]


class OrcArms(C.Structure):
    _fields_ = [("A", f64 * (MAXK * MAXD * MAXD)), ("Ainv", f64 * (MAXK * MAXD * MAXD)),
                ("b", f64 * (MAXK * MAXD)), ("theta", f64 * (MAXK * MAXD)),
                ("rbar", f64 * MAXK), ("ebar", f64 * MAXK), ("n", u32 * MAXK),
                ("active", C.c_uint8 * MAXK)]


class OrcRecord(C.Structure):
    _fields_ = [("arm", C.POINTER(C.c_uint8)), ("near_tie", C.POINTER(C.c_uint8)),
                ("reward", C.POINTER(f64)), ("edp", C.POINTER(f64)), ("energy", C.POINTER(f64)),
                ("tpot", C.POINTER(f64)), ("ttft", C.POINTER(f64)), ("scores", C.POINTER(f64)),
                ("x", C.POINTER(f64)), ("n_active", C.POINTER(u32)),
                ("active_mask", C.POINTER(u32)), ("backlog", C.POINTER(u32)), ("gap", C.POINTER(f64))]


class OrcInject(C.Structure):
    _fields_ = [("x", C.POINTER(f64)), ("edp", C.POINTER(f64)), ("reward", C.POINTER(f64)),
                ("rows", C.POINTER(u32)), ("resp", C.POINTER(f64))]


FREE = 255

DES_RMAX, DES_QMAX, DES_OVER = 128, 512, 0.004


class OrcDesReq(C.Structure):
    _fields_ = [("arr", f64), ("ctx", u32), ("gen", u32), ("tmpl", u32), ("pad", u32)]


class OrcDesSlot(C.Structure):
    _fields_ = [("arr", f64), ("ctx", u32), ("gen", u32), ("done", u32), ("pre", u32), ("used", u32),
                ("pad", u32)]


class OrcDes(C.Structure):
    """ENV.md §7 ENV-S: one tuner's discrete-event server (SPEC inference_sim)."""
    _fields_ = [("clock", f64), ("q", OrcDesReq * DES_QMAX), ("qhead", u32), ("qlen", u32), ("nrun", u32),
                ("kv", u32), ("dropped", u32), ("pad", u32), ("run", OrcDesSlot * DES_RMAX),
                ("store", u32 * 16), ("snap", u32 * 8)]


class OrcDesOut(C.Structure):
    _fields_ = [("E", f64), ("tpot", f64), ("ttft", f64), ("edp", f64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.orc_philox4x32_10.argtypes = [C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]
        L.orc_trace_rows.argtypes = [C.POINTER(OrcConfig), u32, u32, u32, C.POINTER(u32)]
        L.orc_context.argtypes = [C.POINTER(OrcConfig), C.POINTER(u32), C.POINTER(f64)]
        L.orc_env_response.argtypes = [C.POINTER(OrcConfig), C.POINTER(u32), u32, C.POINTER(f64)]
        L.orc_closed_next.argtypes = [C.POINTER(OrcConfig), C.POINTER(u32), u32, u32]
        L.orc_closed_next.restype = u32
        L.orc_step_record.argtypes = [C.POINTER(OrcConfig), C.POINTER(u32), C.POINTER(OrcStepRec)]
        L.orc_response.argtypes = [C.POINTER(OrcConfig), C.POINTER(OrcStepRec), u32, C.POINTER(f64)]
        L.orc_median.argtypes = [C.POINTER(f64), u32]
        L.orc_median.restype = f64
        L.orc_tree128.argtypes = [C.POINTER(f64)]
        L.orc_tree128.restype = f64
        L.orc_invert.argtypes = [u32, C.POINTER(f64), C.POINTER(f64)]
        L.orc_solve.argtypes = [u32, C.POINTER(f64), C.POINTER(f64), C.POINTER(f64)]
        L.orc_run_tuner.argtypes = [C.POINTER(OrcConfig), C.POINTER(OrcTuner), u32,
                                    C.POINTER(C.c_uint8), C.POINTER(OrcStats), C.POINTER(OrcArms),
                                    C.POINTER(OrcRecord)]
        L.orc_run_batch.argtypes = [C.POINTER(OrcConfig), C.POINTER(OrcTuner), u32, u32, C.c_int,
                                    C.POINTER(OrcStats)]
        L.orc_run_tuner_ex.argtypes = [C.POINTER(OrcConfig), C.POINTER(OrcTuner), u32,
                                       C.POINTER(C.c_uint8), C.POINTER(OrcInject),
                                       C.POINTER(OrcStats), C.POINTER(OrcArms), C.POINTER(OrcRecord)]
        L.orc_reward.argtypes = [f64, C.POINTER(f64), u32, f64, f64]
        L.orc_reward.restype = f64
        L.orc_prototype.argtypes = [C.POINTER(OrcConfig), u32, u32]
        L.orc_prototype.restype = u32
        L.orc_sweep.argtypes = [C.POINTER(OrcConfig), u32, u32, u32, C.POINTER(f64), C.POINTER(f64),
                                C.POINTER(u32), C.POINTER(f64), C.POINTER(C.c_uint8)]
        L.orc_argmin.argtypes = [C.POINTER(f64), u32, u32]
        L.orc_argmin.restype = u32
        L.orc_stat_anchor.argtypes = [C.POINTER(OrcConfig), C.POINTER(u32), C.POINTER(f64),
                                      C.POINTER(C.c_uint8)]
        L.orc_stat_anchor.restype = u32
        L.orc_refine_window.argtypes = [C.POINTER(OrcConfig), u32, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)]
        L.orc_refine_window.restype = u32
        L.orc_des_init.argtypes = [C.POINTER(OrcDes)]
        L.orc_des_push.argtypes = [C.POINTER(OrcDes), C.POINTER(OrcConfig), f64, u32, u32, u32]
        L.orc_des_push.restype = C.c_int
        L.orc_des_run.argtypes = [C.POINTER(OrcDes), C.POINTER(OrcConfig), u32, f64, C.POINTER(OrcDesOut)]
        L.orc_des_window.argtypes = [C.POINTER(OrcDes), C.POINTER(OrcConfig), u32, u32, u32, C.POINTER(OrcDesOut)]
        L.orc_sizeof.argtypes = [C.c_int]
        L.orc_sizeof.restype = u32
        for i, s in enumerate([OrcConfig, OrcTuner, OrcStats, OrcArms, OrcStepRec, OrcRecord,
                               OrcInject, OrcDes]):
            assert L.orc_sizeof(i) == C.sizeof(s), (s.__name__, L.orc_sizeof(i), C.sizeof(s))
        _lib = L
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def make_config(cfg: dict) -> OrcConfig:
    oc = OrcConfig()
    for name, ct in OrcConfig._fields_:
        if name.startswith("pad"):
            continue
        v = cfg[name]
        if hasattr(ct, "_length_"):
            arr = getattr(oc, name)
            for i, e in enumerate(v):
                arr[i] = e
        else:
            setattr(oc, name, v)
    return oc


def stat_anchor(cfg: dict, n, ebar, extreme=None):
    """ENV.md §4.11 statistical anchor (arm index, or None)."""
    K = cfg["n_arms"]
    n = np.ascontiguousarray(n, dtype=np.uint32)
    e = np.ascontiguousarray(ebar, dtype=np.float64)
    x = np.zeros(K, np.uint8) if extreme is None else np.ascontiguousarray(extreme, dtype=np.uint8)
    a = lib().orc_stat_anchor(C.byref(make_config(cfg)), _ptr(n, u32), _ptr(e, f64), _ptr(x, C.c_uint8))
    return None if a == 0xFFFFFFFF else int(a)


def refine_window(cfg: dict, anchor: int, extreme=None) -> np.ndarray:
    """ENV.md §4.11 refined action space around arm `anchor` (uint8 mask [K])."""
    K = cfg["n_arms"]
    x = np.zeros(K, np.uint8) if extreme is None else np.ascontiguousarray(extreme, dtype=np.uint8)
    out = np.zeros(K, np.uint8)
    lib().orc_refine_window(C.byref(make_config(cfg)), anchor, _ptr(x, C.c_uint8), _ptr(out, C.c_uint8))
    return out


def make_tuner(trace_id=0, alpha0=1.0, ext_reward_threshold=-1.2, hist_k=1.0) -> OrcTuner:
    return OrcTuner(trace_id=int(trace_id), pad=0, alpha0=float(alpha0),
                    ext_reward_threshold=float(ext_reward_threshold), hist_k=float(hist_k))


def tuner_from(cfg: dict, **kw) -> OrcTuner:
    d = dict(trace_id=0, alpha0=cfg["alpha0"], ext_reward_threshold=cfg["ext_reward_threshold"],
             hist_k=cfg["hist_k"])
    d.update(kw)
    return make_tuner(**d)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c, u32), _ptr(k, u32), _ptr(out, u32))
    return out


def trace_rows(cfg: dict, trace_id: int, t0: int, n: int) -> np.ndarray:
    oc = make_config(cfg)
    out = np.zeros((n, 12), dtype=np.uint32)
    lib().orc_trace_rows(C.byref(oc), trace_id, t0, n, _ptr(out, u32))
    return out


def context(cfg: dict, row) -> np.ndarray:
    oc = make_config(cfg)
    r = np.ascontiguousarray(row, dtype=np.uint32)
    x = np.zeros(7)
    lib().orc_context(C.byref(oc), _ptr(r, u32), _ptr(x, f64))
    return x


def closed_next(cfg: dict, row, q: int, f_mhz: int) -> int:
    """ENV.md §6: backlog carried out of a window (row without the carried-in q) run at f_mhz."""
    oc = make_config(cfg)
    r = np.ascontiguousarray(row, dtype=np.uint32)
    return int(lib().orc_closed_next(C.byref(oc), _ptr(r, u32), int(q), int(f_mhz)))


def env_response(cfg: dict, row, f_mhz: int):
    oc = make_config(cfg)
    r = np.ascontiguousarray(row, dtype=np.uint32)
    out = np.zeros(4)
    lib().orc_env_response(C.byref(oc), _ptr(r, u32), int(f_mhz), _ptr(out, f64))
    return tuple(float(v) for v in out)   # E, TPOT, TTFT, EDP


RECORD_FIELDS = ["x", "g", "invIm", "invAm", "wIm", "nT", "nE", "baseE", "baseEDP", "I", "P"]


def step_record(cfg: dict, row) -> dict:
    """ENV.md §3.2 per-window record (x, g, invIm, invAm, wIm, nT, nE, baseE, baseEDP, I, P)."""
    oc = make_config(cfg)
    r = np.ascontiguousarray(row, dtype=np.uint32)
    rec = OrcStepRec()
    lib().orc_step_record(C.byref(oc), _ptr(r, u32), C.byref(rec))
    out = {n: getattr(rec, n) for n in RECORD_FIELDS}
    out["x"] = np.array(list(rec.x))
    return out


def step_records(cfg: dict, trace_id: int, t0: int, n: int) -> np.ndarray:
    """Records for steps [t0, t0+n) as a (n, 16) float64 view-compatible array (128 B each)."""
    rows = trace_rows(cfg, trace_id, t0, n)
    oc = make_config(cfg)
    out = np.zeros((n, 16), dtype=np.float64)
    rec = OrcStepRec()
    for i in range(n):
        lib().orc_step_record(C.byref(oc), _ptr(np.ascontiguousarray(rows[i]), u32), C.byref(rec))
        C.memmove(out[i].ctypes.data, C.addressof(rec), 128)
    return out


def median(values) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return float(lib().orc_median(_ptr(v, f64), len(v)))


def tree128(values) -> float:
    v = np.zeros(128)
    v[: len(values)] = values
    return float(lib().orc_tree128(_ptr(v, f64)))


def invert(A) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    d = A.shape[0]
    out = np.zeros((d, d))
    rc = lib().orc_invert(d, _ptr(A, f64), _ptr(out, f64))
    assert rc == 0
    return out


def solve(A, b) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    d = A.shape[0]
    out = np.zeros(d)
    rc = lib().orc_solve(d, _ptr(A, f64), _ptr(b, f64), _ptr(out, f64))
    assert rc == 0
    return out


STATS_FIELDS = [n for n, _ in OrcStats._fields_]


def _stats_dict(s: OrcStats) -> dict:
    return {n: getattr(s, n) for n in STATS_FIELDS}


def reward(edp: float, window, clip_lo=-2.0, clip_hi=2.0) -> float:
    w = np.ascontiguousarray(window, dtype=np.float64)
    return float(lib().orc_reward(float(edp), _ptr(w, f64) if len(w) else None, len(w),
                                  clip_lo, clip_hi))


def run_tuner(cfg: dict, tuner: OrcTuner | None = None, T: int | None = None, follow=None,
              record: bool = False, scores: bool = False, inject: dict | None = None):
    """Run one tuner; returns (stats dict, arms dict, record dict or None).

    ``inject`` = {"x": [T,d], "edp": [T,K] or None, "reward": [T,K] or None} replaces the
    synthetic environment (unit tests of the bandit core); the live controller's environment is
    {"rows": [T,12] snapshot rows, "resp": [T,K,3] measured (E, TPOT, TTFT)}. ``follow[t] == FREE`` leaves
    step t unforced."""
    oc = make_config(cfg)
    tu = tuner if tuner is not None else tuner_from(cfg)
    T = cfg["T"] if T is None else T
    st = OrcStats()
    arms = OrcArms()
    recd = None
    rec_p = None
    fol = None
    if follow is not None:
        fol = np.ascontiguousarray(follow, dtype=np.uint8)
        assert len(fol) >= T
    if record:
        K, d = cfg["n_arms"], cfg["d"]
        recd = {"arm": np.zeros(T, np.uint8), "near_tie": np.zeros(T, np.uint8),
                "reward": np.zeros(T), "edp": np.zeros(T), "energy": np.zeros(T),
                "tpot": np.zeros(T), "ttft": np.zeros(T), "x": np.zeros((T, d)),
                "n_active": np.zeros(T, np.uint32), "active_mask": np.zeros((T, 4), np.uint32),
                "backlog": np.zeros(T, np.uint32), "gap": np.zeros(T)}
        if scores:
            recd["scores"] = np.zeros((T, K))
        rec = OrcRecord()
        for name, ct in OrcRecord._fields_:
            if name in recd:
                base = {"arm": C.c_uint8, "near_tie": C.c_uint8, "n_active": u32,
                        "active_mask": u32, "backlog": u32}.get(name, f64)
                setattr(rec, name, _ptr(recd[name], base))
        rec_p = C.byref(rec)
    inj_p = None
    keep = []
    if inject is not None:
        inj = OrcInject()
        for name in ("x", "edp", "reward", "rows", "resp"):
            v = inject.get(name)
            if v is not None:
                dt, ct = (np.uint32, u32) if name == "rows" else (np.float64, f64)
                a = np.ascontiguousarray(v, dtype=dt)
                keep.append(a)
                setattr(inj, name, _ptr(a, ct))
        inj_p = C.byref(inj)
    rc = lib().orc_run_tuner_ex(C.byref(oc), C.byref(tu), T,
                                _ptr(fol, C.c_uint8) if fol is not None else None, inj_p,
                                C.byref(st), C.byref(arms), rec_p)
    assert rc == 0, rc
    K, d = cfg["n_arms"], cfg["d"]
    A = np.ctypeslib.as_array(arms.A).reshape(MAXK, MAXD, MAXD)[:K, :d, :d].copy()
    Ainv = np.ctypeslib.as_array(arms.Ainv).reshape(MAXK, MAXD, MAXD)[:K, :d, :d].copy()
    ad = {"A": A, "Ainv": Ainv,
          "b": np.ctypeslib.as_array(arms.b).reshape(MAXK, MAXD)[:K, :d].copy(),
          "theta": np.ctypeslib.as_array(arms.theta).reshape(MAXK, MAXD)[:K, :d].copy(),
          "rbar": np.ctypeslib.as_array(arms.rbar)[:K].copy(),
          "ebar": np.ctypeslib.as_array(arms.ebar)[:K].copy(),
          "n": np.ctypeslib.as_array(arms.n)[:K].copy(),
          "active": np.ctypeslib.as_array(arms.active)[:K].copy()}
    return _stats_dict(st), ad, recd


def run_batch(cfg: dict, params: dict, T: int, threads: int = 0):
    """Free-running batch on a pthread pool; returns a list of stats dicts."""
    oc = make_config(cfg)
    n = len(params["trace_id"])
    tuners = (OrcTuner * n)()
    for i in range(n):
        tuners[i] = make_tuner(params["trace_id"][i], params["alpha0"][i],
                               params["ext_reward_threshold"][i], params["hist_k"][i])
    stats = (OrcStats * n)()
    rc = lib().orc_run_batch(C.byref(oc), tuners, n, T, threads, stats)
    assert rc == 0, rc
    return [_stats_dict(stats[i]) for i in range(n)]


def prototype(cfg: dict, trace_id: int, t: int) -> int:
    """ENV.md §2.2: the Table-1 prototype index of window t of trace trace_id."""
    return int(lib().orc_prototype(C.byref(make_config(cfg)), trace_id, t))


def new_sweep(cfg: dict) -> dict:
    """Zeroed ENV.md §5 accumulators for one trace."""
    K = cfg["n_arms"]
    return {"S": np.zeros((K, 3)), "SP": np.zeros((5, K)), "NP": np.zeros(5, np.uint32), "O": np.zeros(2)}


def sweep(cfg: dict, trace_id: int, t0: int, n: int, acc: dict | None = None, best: bool = False):
    """ENV.md §5 over windows [t0, t0+n) of one trace, accumulating into ``acc`` (new if None).
    Returns (acc, per-window oracle arm k° or None)."""
    acc = new_sweep(cfg) if acc is None else acc
    b = np.zeros(n, np.uint8) if best else None
    lib().orc_sweep(C.byref(make_config(cfg)), trace_id, t0, n, _ptr(acc["S"], f64), _ptr(acc["SP"], f64),
                    _ptr(acc["NP"], u32), _ptr(acc["O"], f64), _ptr(b, C.c_uint8) if best else None)
    return acc, b


def offline_arm(values) -> int:
    """Smallest index minimising ``values`` (ENV.md §5 k_off)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    return int(lib().orc_argmin(_ptr(v, f64), len(v), 1))


class DesServer:
    """ENV.md §7 ENV-S server (test infrastructure): push requests, run windows, read the snapshot."""

    def __init__(self, cfg: dict):
        self.oc = make_config(cfg)
        self.s = OrcDes()
        lib().orc_des_init(C.byref(self.s))

    def push(self, arr: float, ctx: int, gen: int, tmpl: int) -> bool:
        """Queue a request; False if it was dropped (does not fit the KV cache or a full queue)."""
        return lib().orc_des_push(C.byref(self.s), C.byref(self.oc), float(arr), ctx, gen, tmpl) == 0

    def run(self, f_mhz: int, t_end: float) -> dict:
        o = OrcDesOut()
        lib().orc_des_run(C.byref(self.s), C.byref(self.oc), int(f_mhz), float(t_end), C.byref(o))
        return {"E": o.E, "tpot": o.tpot, "ttft": o.ttft, "edp": o.edp}

    def window(self, trace_id: int, t: int, f_mhz: int) -> dict:
        o = OrcDesOut()
        lib().orc_des_window(C.byref(self.s), C.byref(self.oc), trace_id, t, int(f_mhz), C.byref(o))
        return {"E": o.E, "tpot": o.tpot, "ttft": o.ttft, "edp": o.edp}

    @property
    def snap(self) -> list:
        """[waiting, running, prefill, decode, iterations, kv_used, hits, misses] of the last window."""
        return list(self.s.snap)

    @property
    def state(self) -> dict:
        run = [self.s.run[k] for k in range(DES_RMAX) if self.s.run[k].used]
        return {"clock": self.s.clock, "qlen": self.s.qlen, "nrun": self.s.nrun, "kv": self.s.kv,
                "dropped": self.s.dropped, "running": [(r.ctx, r.gen, r.done, r.pre) for r in run]}
