"""ctypes binding of include/agft.h — argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``libagft.so``; this module
only converts Python configs / torch tensors into the C structs and pointers the
ABI takes. There is no CPU fallback: if the library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AGFT_LIB_PATH") or os.path.join(HERE, "libagft.so")   # override: A/B builds

ABI_VERSION = 9
RECORD_BYTES = 128
ROW_WORDS = 12
NO_RECORD = 0xFFFFFFFF
MAX_ARMS = 128

u32, u64, f64, vp = C.c_uint32, C.c_uint64, C.c_double, C.c_void_p


class AgftGrid(C.Structure):
    _fields_ = [("f_min_mhz", u32), ("f_step_mhz", u32), ("n_arms", u32), ("f_max_hw_mhz", u32)]


class AgftPrune(C.Structure):
    _fields_ = [("enable", u32), ("extreme_round_limit", u32), ("extreme_min_samples", u32),
                ("historical_min_round", u32), ("historical_min_samples", u32), ("pad", u32),
                ("cascade_fraction", f64)]


class AgftPolicy(C.Structure):
    _fields_ = [("tau", f64), ("clip_lo", f64), ("clip_hi", f64), ("tie_rel", f64),
                ("median_window", u32), ("pad", u32)]


class AgftEnv(C.Structure):
    _fields_ = [(n, f64) for n in ("window_s", "p_idle", "k_lin", "k_cube", "u_floor", "u_max",
                                   "c_prefill", "c_decode", "beta", "sigma_e", "sigma_t")]


class AgftTraceCfg(C.Structure):
    _fields_ = [("lambda0", f64), ("burst_mult", f64), ("t_iter0", f64), ("t_iter1", f64),
                ("e2e0", f64), ("tau_ref", f64),
                ("seg_steps", u32), ("steps_per_hour", u32), ("burst_steps", u32), ("burst_p32", u32),
                ("cap", u32), ("kv_total", u32), ("pattern_mode", u32), ("pad", u32),
                ("ctx_lo", u32 * 5), ("ctx_hi", u32 * 5), ("gen_lo", u32 * 5), ("gen_hi", u32 * 5),
                ("weight", u32 * 5), ("pad2", u32),
                ("conc_mult", f64 * 5), ("hit_rate", f64 * 5), ("knot", f64 * 24)]


class AgftPhase(C.Structure):
    _fields_ = [("enable", u32), ("window", u32), ("delta", f64), ("lambda_", f64)]


class AgftRefine(C.Structure):
    _fields_ = [("enable", u32), ("period", u32), ("mature", u32), ("min_samples", u32),
                ("half_mhz", u32), ("step_mhz", u32)]


class AgftClosed(C.Structure):
    _fields_ = [("enable", u32), ("q_max", u32)]


class AgftConfig(C.Structure):
    _fields_ = [("abi_version", u32), ("n_tuners", u32), ("d", u32), ("n_traces", u32),
                ("trace_base", u32), ("record_slots", u32), ("kernel_policy", u32), ("pad0", u32),
                ("grid", AgftGrid), ("prune", AgftPrune), ("policy", AgftPolicy), ("env", AgftEnv),
                ("trace", AgftTraceCfg), ("norm_lo", f64 * 7), ("norm_hi", f64 * 7), ("env_seed", u64),
                ("phase", AgftPhase), ("refine", AgftRefine), ("pad1", u32), ("closed", AgftClosed)]


PARAMS_DTYPE = np.dtype([("trace_id", "<u4"), ("record_slot", "<u4"), ("alpha0", "<f8"),
                         ("extreme_reward_threshold", "<f8"), ("historical_k", "<f8")])
STATS_DTYPE = np.dtype([("traj_hash", "<u8"), ("sum_active", "<u8"),
                        ("steps", "<u4"), ("last_arm", "<u4"), ("n_active", "<u4"),
                        ("n_pruned_extreme", "<u4"), ("n_pruned_hist", "<u4"),
                        ("n_pruned_cascade", "<u4"), ("near_tie_steps", "<u4"), ("flags", "<u4"),
                        ("sum_energy", "<f8"), ("sum_tpot", "<f8"), ("sum_ttft", "<f8"),
                        ("sum_edp", "<f8"), ("sum_reward", "<f8"), ("base_energy", "<f8"),
                        ("base_edp", "<f8"), ("exploit_steps", "<u4"), ("ph_alarms", "<u4"),
                        ("first_exploit_t", "<u4"), ("phase", "<u4"), ("n_refine", "<u4"),
                        ("last_anchor", "<u4")])
assert PARAMS_DTYPE.itemsize == 32 and STATS_DTYPE.itemsize == 128

STATUS = {0: "ok", -1: "invalid argument", -2: "invalid frequency grid", -3: "empty arm set",
          -4: "context dimension out of range", -5: "non-finite or out-of-range coefficient",
          -6: "workspace too small or misaligned", -7: "step counter mismatch", -8: "CUDA error",
          -9: "no sm_100 device"}

# name → (restype, argtypes); the export list tests/test_abi.py checks against include/agft.h
PROTOTYPES = {
    "agft_validate": (C.c_int, [C.POINTER(AgftConfig)]),
    "agft_struct_size": (u32, [C.c_int]),
    "agft_workspace_bytes": (C.c_size_t, [C.POINTER(AgftConfig)]),
    "agft_create": (C.c_int, [C.POINTER(AgftConfig), vp, vp, C.c_size_t, vp, C.POINTER(vp)]),
    "agft_reset": (C.c_int, [vp]),
    "agft_attach": (C.c_int, [C.POINTER(AgftConfig), vp, C.c_size_t, vp, u32, u32, C.POINTER(vp)]),
    "agft_trace_generate": (C.c_int, [vp, u32, u32, vp, vp]),
    "agft_step": (C.c_int, [vp, vp, vp]),
    "agft_select": (C.c_int, [vp, vp, vp]),
    "agft_observe": (C.c_int, [vp, vp]),
    "agft_scores": (C.c_int, [vp, vp, vp, vp]),
    "agft_replay": (C.c_int, [vp, vp, u32, u32, vp, vp]),
    "agft_replay_raw": (C.c_int, [vp, vp, vp, u32, u32, vp, vp]),
    "agft_stats": (C.c_int, [vp, vp]),
    "agft_export_arms": (C.c_int, [vp, u32, vp, vp, vp, vp, vp, vp, vp]),
    "agft_get_step": (C.c_int, [vp, C.POINTER(u32)]),
    "agft_get_counters": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
    "agft_run": (C.c_int, [C.POINTER(AgftConfig), vp, vp, u32, u32, vp, C.c_size_t, vp, C.c_size_t,
                           vp, vp, vp]),
    "agft_sweep": (C.c_int, [vp, vp, u32, u32, vp, vp, vp, vp, vp]),
    "agft_regret": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
    "agft_destroy": (C.c_int, [vp]),
    "agft_status_string": (C.c_char_p, [C.c_int]),
    "agft_kernel_launches": (C.c_uint64, []),
    "agft_profile_start": (C.c_int, [vp, C.c_int]),
    "agft_profile_read": (C.c_int, [vp, vp]),
    "agft_timeline": (C.c_int, [vp, vp, C.c_uint64]),
    "agft_occupancy": (C.c_int, [C.POINTER(AgftConfig), C.c_int, C.POINTER(u32)]),
}

# agft_profile slots (include/agft.h): the replay classes, then the classification and refinement passes
PROFILE_SLOTS = ("wide", "seg_g16", "seg_g8", "seg_g4", "solo", "seg_g32", "classify", "refine")


class AgftProfile(C.Structure):
    _fields_ = [("tuner_steps", u64 * 8), ("active_arm_steps", u64 * 8), ("kernel_ms", f64 * 8),
                ("launches", u32 * 8)]

_lib = None


class AgftError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {code} ({STATUS.get(code, 'unknown')})")
        self.code = code


def lib():
    """Load libagft.so (built in-tree by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing — run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        sizes = (C.sizeof(AgftConfig), PARAMS_DTYPE.itemsize, STATS_DTYPE.itemsize)
        for i, sz in enumerate(sizes):
            if L.agft_struct_size(i) != sz:
                raise RuntimeError(f"ABI mirror mismatch for struct {i}: C {L.agft_struct_size(i)} vs {sz}")
        _lib = L
    return _lib


def check(fn: str, code: int):
    if code != 0:
        raise AgftError(fn, code)


def make_config(cfg: dict, n_tuners: int | None = None, n_traces: int | None = None,
                trace_base: int = 0, record_slots: int = 0, policy: int = 0) -> AgftConfig:
    """Marshal a named-config dict (agft_inputs.configs) into the C agft_config."""
    c = AgftConfig()
    c.abi_version = ABI_VERSION
    c.kernel_policy = policy
    c.n_tuners = cfg["n_tuners"] if n_tuners is None else n_tuners
    c.d = cfg["d"]
    c.n_traces = cfg["n_traces"] if n_traces is None else n_traces
    c.trace_base = trace_base
    c.record_slots = record_slots
    c.grid = AgftGrid(cfg["f_min_mhz"], cfg["f_step_mhz"], cfg["n_arms"], cfg["f_max_hw_mhz"])
    c.prune = AgftPrune(cfg["prune_enable"], cfg["ext_round_limit"], cfg["ext_min_samples"],
                        cfg["hist_min_round"], cfg["hist_min_samples"], 0, cfg["cascade_fraction"])
    c.policy = AgftPolicy(cfg["tau"], cfg["clip_lo"], cfg["clip_hi"], cfg["tie_rel"],
                          cfg["median_window"], 0)
    c.env = AgftEnv(cfg["W"], cfg["p_idle"], cfg["k_lin"], cfg["k_cube"], cfg["u_floor"],
                    cfg["u_max"], cfg["c_p"], cfg["c_d"], cfg["beta"], cfg["sigma_e"],
                    cfg["sigma_t"])
    t = c.trace
    for n in ("lambda0", "burst_mult", "t_iter0", "t_iter1", "e2e0", "tau_ref", "seg_steps",
              "steps_per_hour", "burst_steps", "burst_p32", "cap", "kv_total", "pattern_mode"):
        setattr(t, n, cfg[n])
    for n in ("ctx_lo", "ctx_hi", "gen_lo", "gen_hi", "weight", "conc_mult", "hit_rate", "knot"):
        arr = getattr(t, n)
        for i, v in enumerate(cfg[n]):
            arr[i] = v
    for i in range(7):
        c.norm_lo[i] = cfg["norm_lo"][i]
        c.norm_hi[i] = cfg["norm_hi"][i]
    c.env_seed = cfg["seed"]
    c.phase = AgftPhase(cfg.get("ph_enable", 0), cfg.get("ph_window", 50), cfg.get("ph_delta", 0.005),
                        cfg.get("ph_lambda", 0.25))
    c.refine = AgftRefine(cfg.get("rf_enable", 0), cfg.get("rf_period", 25), cfg.get("rf_mature", 100),
                          cfg.get("rf_min_samples", 4), cfg.get("rf_half_mhz", 150), cfg.get("rf_step_mhz", 15))
    c.closed = AgftClosed(cfg.get("cl_enable", 0), cfg.get("cl_q_max", 256))
    return c


def make_params(params: dict, record_slot=None) -> np.ndarray:
    """Per-tuner params (agft_inputs.tuner_params output) → agft_tuner_params[N] bytes."""
    n = len(params["trace_id"])
    out = np.zeros(n, dtype=PARAMS_DTYPE)
    out["trace_id"] = params["trace_id"]
    out["alpha0"] = params["alpha0"]
    out["extreme_reward_threshold"] = params["ext_reward_threshold"]
    out["historical_k"] = params["hist_k"]
    out["record_slot"] = NO_RECORD if record_slot is None else record_slot
    return out
