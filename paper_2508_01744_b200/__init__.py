"""B200-native AGFT hot path: a batched replay of LinUCB GPU-frequency tuners.

The Python layer marshals arguments into the C ABI of ``include/agft.h``
(``libagft.so``, hand-written sm_100a kernels). PyTorch provides device memory,
streams and process groups only. Names follow the ABI: ``agft_create``,
``agft_trace_generate``, ``agft_step``, ``agft_replay``, ``agft_stats``,
``agft_export_arms``, ``agft_run``, ``agft_sweep``, ``agft_regret``, ``agft_destroy``, and the
live two-phase step ``agft_select`` / ``agft_observe``.
``TunerBatch`` bundles them.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import (NO_RECORD, PARAMS_DTYPE, RECORD_BYTES, ROW_WORDS, STATS_DTYPE, AgftError,
                   make_config, make_params)

__all__ = ["agft_workspace_bytes", "agft_create", "agft_reset", "agft_trace_generate", "agft_step", "agft_replay",
           "agft_select", "agft_observe", "agft_scores", "agft_replay_raw", "agft_attach",
           "agft_stats", "agft_export_arms", "agft_get_step", "agft_get_counters", "agft_run", "agft_sweep",
           "agft_regret",
           "agft_destroy", "SweepSums",
           "TunerBatch", "record_slot_count", "make_config", "make_params", "PARAMS_DTYPE", "STATS_DTYPE", "NO_RECORD",
           "RECORD_BYTES", "ROW_WORDS", "AgftError", "lib_path"]


def lib_path() -> str:
    return _abi.LIB_PATH


def _p(t):
    """Device (or host) pointer of a torch tensor / numpy array, or None."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _on_device(fn):
    """Run a TunerBatch method with its device current: the library launches on the current
    device and creates its side streams there."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **k):
        import torch
        with torch.cuda.device(self.device):
            return fn(self, *a, **k)
    return wrapped


def agft_workspace_bytes(cfg_c: _abi.AgftConfig) -> int:
    return int(_abi.lib().agft_workspace_bytes(C.byref(cfg_c)))


def agft_create(cfg_c, d_params, workspace, stream=None) -> int:
    h = C.c_void_p()
    _abi.check("agft_create", _abi.lib().agft_create(C.byref(cfg_c), _p(d_params), _p(workspace),
                                                      workspace.numel() * workspace.element_size(),
                                                      _stream(stream), C.byref(h)))
    return h.value


def agft_attach(cfg_c, workspace, t, sweep_t=0, stream=None) -> int:
    h = C.c_void_p()
    _abi.check("agft_attach", _abi.lib().agft_attach(C.byref(cfg_c), _p(workspace),
                                                      workspace.numel() * workspace.element_size(),
                                                      _stream(stream), t, sweep_t, C.byref(h)))
    return h.value


def agft_reset(h):
    _abi.check("agft_reset", _abi.lib().agft_reset(h))


def agft_trace_generate(h, t0, n_steps, records, raw=None):
    _abi.check("agft_trace_generate", _abi.lib().agft_trace_generate(h, t0, n_steps, _p(records), _p(raw)))


def agft_step(h, records, chosen=None):
    _abi.check("agft_step", _abi.lib().agft_step(h, _p(records), _p(chosen)))


def agft_select(h, rows, chosen):
    _abi.check("agft_select", _abi.lib().agft_select(h, _p(rows), _p(chosen)))


def agft_observe(h, resp):
    _abi.check("agft_observe", _abi.lib().agft_observe(h, _p(resp)))


def agft_scores(h, rows, scores, chosen=None):
    _abi.check("agft_scores", _abi.lib().agft_scores(h, _p(rows), _p(scores), _p(chosen)))


def agft_replay(h, records, t0, n_steps, traj=None, gap=None):
    _abi.check("agft_replay", _abi.lib().agft_replay(h, _p(records), t0, n_steps, _p(traj), _p(gap)))


def agft_replay_raw(h, records, raw, t0, n_steps, traj=None, gap=None):
    _abi.check("agft_replay_raw", _abi.lib().agft_replay_raw(h, _p(records), _p(raw), t0, n_steps, _p(traj),
                                                              _p(gap)))


def agft_stats(h, out):
    _abi.check("agft_stats", _abi.lib().agft_stats(h, _p(out)))


def agft_export_arms(h, tuner, ainv=None, b=None, theta=None, n=None, rbar=None, ebar=None, mask=None):
    _abi.check("agft_export_arms", _abi.lib().agft_export_arms(h, tuner, _p(ainv), _p(b), _p(theta),
                                                                _p(n), _p(rbar), _p(ebar), _p(mask)))


def agft_get_step(h) -> int:
    t = C.c_uint32()
    _abi.check("agft_get_step", _abi.lib().agft_get_step(h, C.byref(t)))
    return t.value


def agft_get_counters(h) -> tuple[int, int, int]:
    """(step counter t, sweep counter, live_pending) of a handle: what a checkpoint stores."""
    t, sw, lp = C.c_uint32(), C.c_uint32(), C.c_uint32()
    _abi.check("agft_get_counters", _abi.lib().agft_get_counters(h, C.byref(t), C.byref(sw), C.byref(lp)))
    return t.value, sw.value, lp.value


def agft_profile_start(h, serialize: bool = False):
    """Start per-class accounting; serialize=True runs each class alone (per-kernel event times)."""
    _abi.check("agft_profile_start", _abi.lib().agft_profile_start(h, int(bool(serialize))))


def agft_profile_read(h) -> dict:
    """Per-class tuner-steps, Σ K_act, event time and launches since agft_profile_start (synchronises)."""
    p = _abi.AgftProfile()
    _abi.check("agft_profile_read", _abi.lib().agft_profile_read(h, C.byref(p)))
    return {name: {"tuner_steps": int(p.tuner_steps[i]), "active_arm_steps": int(p.active_arm_steps[i]),
                   "kernel_ms": float(p.kernel_ms[i]), "launches": int(p.launches[i])}
            for i, name in enumerate(_abi.PROFILE_SLOTS)}


def agft_timeline(h, buf, cap_records: int = 0):
    """Per-warp scheduling records of the replay-class launches into the int64 device tensor `buf`
    (8 × (1 + 3 × cap_records) bytes); buf=None turns recording off (include/agft.h)."""
    _abi.check("agft_timeline", _abi.lib().agft_timeline(h, _p(buf) if buf is not None else None,
                                                         int(cap_records)))


def agft_occupancy(cfg_c, slot: int) -> int:
    """Resident tuners per SM of replay class `slot` (_abi.PROFILE_SLOTS order) for this config."""
    v = C.c_uint32()
    _abi.check("agft_occupancy", _abi.lib().agft_occupancy(C.byref(cfg_c), slot, C.byref(v)))
    return v.value


def agft_sweep(h, records, t0, n_steps, S, SP, NP, O, best=None):
    _abi.check("agft_sweep", _abi.lib().agft_sweep(h, _p(records), t0, n_steps, _p(S), _p(SP), _p(NP), _p(O),
                                                    _p(best)))


def agft_regret(h, S, SP, NP, O, koff, regret=None):
    _abi.check("agft_regret", _abi.lib().agft_regret(h, _p(S), _p(SP), _p(NP), _p(O), _p(koff), _p(regret)))


class SweepSums:
    """Caller-owned ENV.md §5 accumulators for every local trace (zeroed device tensors)."""

    def __init__(self, n_traces: int, n_arms: int, device):
        import torch
        self.S = torch.zeros((n_traces, n_arms, 3), dtype=torch.float64, device=device)
        self.SP = torch.zeros((n_traces, 5, n_arms), dtype=torch.float64, device=device)
        self.NP = torch.zeros((n_traces, 5), dtype=torch.int32, device=device)
        self.O = torch.zeros((n_traces, 2), dtype=torch.float64, device=device)
        self.koff = torch.zeros((n_traces, 6), dtype=torch.uint8, device=device)

    def host(self) -> dict:
        return {"S": self.S.cpu().numpy(), "SP": self.SP.cpu().numpy(),
                "NP": self.NP.cpu().numpy().view(np.uint32), "O": self.O.cpu().numpy(),
                "koff": self.koff.cpu().numpy()}


def agft_run(cfg_c, h_params, d_params_buf, n_steps, chunk_steps, workspace, scratch, d_stats_buf,
             h_stats, stream=None):
    _abi.check("agft_run", _abi.lib().agft_run(
        C.byref(cfg_c), _p(h_params), _p(d_params_buf), n_steps, chunk_steps, _p(workspace),
        workspace.numel() * workspace.element_size(), _p(scratch),
        scratch.numel() * scratch.element_size(), _p(d_stats_buf), _p(h_stats), _stream(stream)))


def agft_destroy(h):
    _abi.check("agft_destroy", _abi.lib().agft_destroy(h))


def record_slot_count(record_slot) -> int:
    """Rows of the trajectory record: 1 + the largest slot that is not NO_RECORD (0 if none)."""
    if record_slot is None:
        return 0
    rs = np.asarray(record_slot, dtype=np.int64)
    return int(np.max(np.where(rs == NO_RECORD, -1, rs), initial=-1) + 1)


class TunerBatch:
    """N tuners on one GPU: owns (torch-allocated) workspace, params and the handle."""

    def __init__(self, cfg: dict, params: dict, device="cuda", record_slot=None, trace_base: int = 0,
                 n_traces: int | None = None, stream=None, policy: int = 0):
        import torch
        self.cfg = cfg
        self.device = torch.device(device)
        self.n = len(params["trace_id"])
        self.n_traces = cfg["n_traces"] if n_traces is None else n_traces
        rec_slots = record_slot_count(record_slot)
        self.record_slots = rec_slots
        self.cfg_c = make_config(cfg, n_tuners=self.n, n_traces=self.n_traces, trace_base=trace_base,
                                 record_slots=rec_slots, policy=policy)
        ws = agft_workspace_bytes(self.cfg_c)
        if ws == 0:
            raise AgftError("agft_workspace_bytes", -1)
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
        host = make_params(params, record_slot)
        self.d_params = torch.from_numpy(host.view(np.uint8)).to(self.device)
        self.stream = stream
        with torch.cuda.device(self.device):
            self.h = agft_create(self.cfg_c, self.d_params, self.workspace,
                                 stream if stream is not None else torch.cuda.current_stream(self.device))

    @_on_device
    def reset(self):
        agft_reset(self.h)

    def checkpoint(self):
        """(workspace bytes on the host, step counter, sweep counter): everything a resume needs
        (S:224).  The tuner parameters live in the workspace.  Refused between agft_select and its
        agft_observe (the pending selection is not part of the state a resume restores)."""
        import torch
        t, sweep_t, pending = agft_get_counters(self.h)
        if pending:
            raise AgftError("checkpoint: a live selection is pending (agft_select without agft_observe)", -7)
        torch.cuda.synchronize(self.device)
        return self.workspace.cpu(), t, sweep_t

    @classmethod
    def resume(cls, cfg: dict, params: dict, state, device="cuda", trace_base: int = 0, n_traces=None,
               record_slot=None, policy: int = 0):
        """A TunerBatch on a copy of a checkpointed workspace, continuing at its step and sweep
        counters.  The tuner parameters come from the workspace (``params`` only sizes the batch)."""
        import torch
        self = cls.__new__(cls)
        self.cfg = cfg
        self.device = torch.device(device)
        self.n = len(params["trace_id"])
        self.n_traces = cfg["n_traces"] if n_traces is None else n_traces
        self.record_slots = record_slot_count(record_slot)
        self.cfg_c = make_config(cfg, n_tuners=self.n, n_traces=self.n_traces, trace_base=trace_base,
                                 record_slots=self.record_slots, policy=policy)
        ws_host, t = state[0], state[1]
        sweep_t = state[2] if len(state) > 2 else 0
        self.workspace = ws_host.to(self.device)
        self.d_params = None
        self.stream = None
        with torch.cuda.device(self.device):
            self.h = agft_attach(self.cfg_c, self.workspace, t, sweep_t, torch.cuda.current_stream(self.device))
        return self

    @property
    def t(self) -> int:
        return agft_get_step(self.h)

    def new_records(self, n_steps: int):
        import torch
        return torch.empty((self.n_traces, n_steps, RECORD_BYTES), dtype=torch.uint8, device=self.device)

    @_on_device
    def generate(self, t0: int, n_steps: int, records=None, raw: bool = False):
        import torch
        records = self.new_records(n_steps) if records is None else records
        rawt = (torch.empty((self.n_traces, n_steps, ROW_WORDS), dtype=torch.int32, device=self.device)
                if raw else None)
        agft_trace_generate(self.h, t0, n_steps, records, rawt)
        return (records, rawt) if raw else records

    @property
    def closed(self) -> bool:
        """ENV-C closed loop (ENV.md §6): replays need the raw rows (agft_replay_raw)."""
        return bool(self.cfg.get("cl_enable", 0))

    @_on_device
    def replay(self, records, t0: int, n_steps: int, record: bool = False, raw=None):
        import torch
        traj = gap = None
        if record and self.record_slots:
            traj = torch.zeros((self.record_slots, n_steps), dtype=torch.uint8, device=self.device)
            gap = torch.zeros((self.record_slots, n_steps), dtype=torch.float64, device=self.device)
        if raw is not None:
            agft_replay_raw(self.h, records, raw, t0, n_steps, traj, gap)
        else:
            agft_replay(self.h, records, t0, n_steps, traj, gap)
        return traj, gap

    @_on_device
    def step(self, records_t):
        import torch
        chosen = torch.empty(self.n, dtype=torch.int32, device=self.device)
        agft_step(self.h, records_t, chosen)
        return chosen

    @_on_device
    def select(self, rows, chosen=None):
        """Live step, first half: rows [n][12] int32 device tensor of MetricsSnapshot counters →
        chosen arm per tuner (int32 [n] device tensor; -1 = frozen tuner)."""
        import torch
        if chosen is None:
            chosen = torch.empty(self.n, dtype=torch.int32, device=self.device)
        agft_select(self.h, rows, chosen)
        return chosen

    @_on_device
    def scores(self, rows):
        """Read-only Eq. 1 scores [n][K] (float64, NaN for pruned arms) at the current step for the
        snapshot rows [n][12] (int32 device tensor), and the arg max per tuner."""
        import torch
        out = torch.empty((self.n, self.cfg["n_arms"]), dtype=torch.float64, device=self.device)
        chosen = torch.empty(self.n, dtype=torch.int32, device=self.device)
        agft_scores(self.h, rows, out, chosen)
        return out, chosen

    @_on_device
    def observe(self, resp):
        """Live step, second half: resp [n][3] float64 device tensor of measured (E J, TPOT s,
        TTFT s) at the selected frequencies."""
        agft_observe(self.h, resp)

    @_on_device
    def run(self, T: int, chunk: int = 4500, record: bool = False):
        """Generate + replay steps [t, T) in chunks; returns recorded traj/gap (host) if asked."""
        import torch
        trajs, gaps = [], []
        rec = raw = None
        t = self.t
        while t < T:
            n = min(chunk, T - t)
            if rec is None or rec.shape[1] != n:
                rec = self.new_records(n)
                raw = (torch.empty((self.n_traces, n, ROW_WORDS), dtype=torch.int32, device=self.device)
                       if self.closed else None)
            agft_trace_generate(self.h, t, n, rec, raw)
            tr, gp = self.replay(rec, t, n, record=record, raw=raw)
            if record and tr is not None:
                trajs.append(tr.cpu())
                gaps.append(gp.cpu())
            t += n
        if record and trajs:
            return torch.cat(trajs, 1).numpy(), torch.cat(gaps, 1).numpy()
        return None, None

    def new_sweep(self) -> SweepSums:
        return SweepSums(self.n_traces, self.cfg["n_arms"], self.device)

    @_on_device
    def sweep(self, records, t0: int, n_steps: int, sums: SweepSums, best: bool = False):
        """ENV.md §5 over windows [t0, t0+n_steps) into ``sums``; returns k° [n_traces][n] if asked."""
        import torch
        b = torch.empty((self.n_traces, n_steps), dtype=torch.uint8, device=self.device) if best else None
        agft_sweep(self.h, records, t0, n_steps, sums.S, sums.SP, sums.NP, sums.O, b)
        return b

    @_on_device
    def regret(self, sums: SweepSums):
        """Table-6 Offline arms into ``sums.koff`` and per-tuner (window, fixed) regret [n][2]."""
        import torch
        out = torch.empty((self.n, 2), dtype=torch.float64, device=self.device)
        agft_regret(self.h, sums.S, sums.SP, sums.NP, sums.O, sums.koff, out)
        return out

    @_on_device
    def stats_tensor(self):
        import torch
        out = torch.empty(self.n * STATS_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        agft_stats(self.h, out)
        return out

    def stats(self) -> np.ndarray:
        return self.stats_tensor().cpu().numpy().view(STATS_DTYPE)

    @_on_device
    def export_arms(self, tuner: int) -> dict:
        import torch
        K, d = self.cfg["n_arms"], self.cfg["d"]
        P = d * (d + 1) // 2
        dev = self.device
        out = {"ainv_packed": torch.empty((K, P), dtype=torch.float64, device=dev),
               "b": torch.empty((K, d), dtype=torch.float64, device=dev),
               "theta": torch.empty((K, d), dtype=torch.float64, device=dev),
               "n": torch.empty(K, dtype=torch.int32, device=dev),
               "rbar": torch.empty(K, dtype=torch.float64, device=dev),
               "ebar": torch.empty(K, dtype=torch.float64, device=dev),
               "mask": torch.empty(4, dtype=torch.int32, device=dev)}
        agft_export_arms(self.h, tuner, out["ainv_packed"], out["b"], out["theta"], out["n"],
                         out["rbar"], out["ebar"], out["mask"])
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["n"] = res["n"].view(np.uint32)
        m = res.pop("mask").view(np.uint32)
        res["active"] = np.array([(m[k // 32] >> (k % 32)) & 1 for k in range(K)], dtype=np.uint8)
        ainv = np.zeros((K, d, d))
        e = 0
        for i in range(d):
            for j in range(i, d):
                ainv[:, i, j] = res["ainv_packed"][:, e]
                ainv[:, j, i] = res["ainv_packed"][:, e]
                e += 1
        res["Ainv"] = ainv
        return res

    def close(self):
        if getattr(self, "h", None):
            agft_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
