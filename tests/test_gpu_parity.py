"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element
on the same seeded inputs. Bit-exact for trace rows, records, trajectories, counters, b,
n, r̄, ē and every stats sum; 1e-9 relative for A⁻¹ and θ (north_star)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from agft_inputs import named_config, tuner_params  # noqa: E402
from paper_2508_01744_b200 import NO_RECORD, TunerBatch, AgftError  # noqa: E402

from _parity import compare_tuner, oracle_tuner  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _cfg(name, **kw):
    c = named_config(name)
    c.update(kw)
    return c


def _run(cfg, T, ids=None, record=None, chunk=4500, params=None, policy=0):
    params = tuner_params(cfg, ids) if params is None else params
    n = len(params["trace_id"])
    rec_slot = None
    if record is not None:
        rec_slot = np.full(n, NO_RECORD, np.uint32)
        for s, i in enumerate(record):
            rec_slot[i] = s
    tb = TunerBatch(dict(cfg, n_tuners=n), params, device="cuda:0", record_slot=rec_slot, policy=policy)
    traj, gap = tb.run(T, chunk=chunk, record=record is not None)
    st = tb.stats()
    return tb, params, st, traj, gap


def _check(cfg, tb, params, st, idx, T, traj=None, slots=None, arms=True, gap=None):
    problems, infos = [], []
    for s, i in enumerate(idx):
        tr = traj[slots[i] if slots else s] if traj is not None else None
        gp = gap[slots[i] if slots else s] if gap is not None else None
        g = tb.export_arms(i) if arms else None
        errs, info = compare_tuner(cfg, params, i, st[i], g, T, tr, gap=gp)
        problems += errs
        infos.append(info)
    assert not problems, "\n".join(problems[:20])
    return infos


# ---------------------------------------------------------------- a0 / a2: trace rows + records
def test_trace_rows_and_records_bitexact_c2():
    cfg = _cfg("C2")
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    rec, raw = tb.generate(0, 4500, raw=True)
    graw = raw.cpu().numpy().view(np.uint32)[0]
    grec = rec.cpu().numpy()[0]
    assert np.array_equal(graw, oracle.trace_rows(cfg, 0, 0, 4500))
    orec = oracle.step_records(cfg, 0, 0, 4500)
    assert np.array_equal(grec.view(np.uint8), orec.view(np.uint8))


@pytest.mark.parametrize("name,t0,n,traces", [
    ("C3", 2000, 500, [0, 1, 2047, 4095]),
    ("C4", 0, 300, [0, 1, 128, 255]),
    ("C4", 107700, 300, [3, 200]),         # end of the 24-h day, diurnal wrap
    ("C5", 53900, 200, [0, 1, 2, 4095]),   # pattern = trace mod 3
])
def test_trace_records_sampled_full_sizes(name, t0, n, traces):
    cfg = _cfg(name)
    tb = TunerBatch(dict(cfg, n_tuners=1), {k: v[:1] for k, v in tuner_params(cfg, [0]).items()},
                    device="cuda:0", n_traces=cfg["n_traces"])
    rec, raw = tb.generate(t0, n, raw=True)
    graw = raw.cpu().numpy().view(np.uint32)
    grec = rec.cpu().numpy()
    for r in traces:
        assert np.array_equal(graw[r], oracle.trace_rows(cfg, r, t0, n)), (name, r)
        assert np.array_equal(grec[r].view(np.uint8), oracle.step_records(cfg, r, t0, n).view(np.uint8)), (name, r)


# ---------------------------------------------------------------- single tuners (C1, C2)
def test_c1_parity():
    cfg = _cfg("C1")
    tb, params, st, traj, gap = _run(cfg, 1000, record=[0])
    _check(cfg, tb, params, st, [0], 1000, traj, gap=gap)


@pytest.mark.parametrize("policy", [0, 1])
def test_c2_parity(policy):
    cfg = _cfg("C2")
    tb, params, st, traj, gap = _run(cfg, 4500, record=[0], policy=policy)
    _check(cfg, tb, params, st, [0], 4500, traj, gap=gap)
    assert st["n_active"][0] < 107                    # pruning really happened


# ---------------------------------------------------------------- batches
@pytest.mark.parametrize("policy", [0, 1])
def test_c3_sampled_parity(policy):
    cfg = _cfg("C3")
    sample = [0, 1, 31, 32, 33, 1000, 2047, 4094, 4095]
    tb, params, st, traj, gap = _run(cfg, 4500, record=sample, policy=policy)
    _check(cfg, tb, params, st, sample, 4500, traj, gap=gap)
    assert np.all(st["steps"] == 4500) and np.all(st["flags"] == 0)


def test_c4_full_size_sampled_parity():
    """BASELINE configs[3] at full size (65,536 tuners × 108,000 steps) in the bench's launch
    configuration; sampled tuners span α, τ_E, k_h and both load patterns."""
    cfg = _cfg("C4")
    sample = [0, 15, 255, 256 + 48, 256 * 77 + 200, 65535]
    tb, params, st, traj, gap = _run(cfg, cfg["T"], record=sample, chunk=4500)
    _check(cfg, tb, params, st, sample, cfg["T"], traj, gap=gap)
    assert np.all(st["steps"] == cfg["T"]) and np.all(st["flags"] == 0)
    assert np.all(st["n_active"] >= 1)


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("kw", [
    dict(n_arms=1),                                   # degenerate single arm
    dict(d=1),
    dict(median_window=1),
    dict(median_window=2),
    dict(median_window=63),
    dict(prune_enable=0),
    dict(n_arms=33, f_step_mhz=45),                   # ragged second slot
    dict(n_arms=96),                                  # three full slots
    dict(hist_min_round=0, hist_min_samples=1),       # aggressive historical pruning
    dict(ext_round_limit=1000, ext_min_samples=1),    # extreme pruning + cascades
    dict(f_min_mhz=1200, n_arms=41),                  # no cascade region
])
@pytest.mark.parametrize("policy", [0, 1])
def test_edge_configs(kw, policy):
    cfg = _cfg("C2", n_tuners=5, n_traces=5, T=700)
    cfg.update(kw)
    ids = list(range(5))
    params = tuner_params(cfg, ids)
    params["alpha0"] = np.array([0.0, 0.3, 1.0, 2.0, 5.0])
    tb, params, st, traj, gap = _run(cfg, 700, params=params, record=ids, chunk=256, policy=policy)
    _check(cfg, tb, params, st, ids, 700, traj, gap=gap)


def test_ragged_tuner_counts_and_shared_trace():
    """N not a multiple of the warps per block; many tuners on one trace (C4-style sharing)."""
    for n in (1, 3, 37):
        cfg = _cfg("C2", n_tuners=n, n_traces=1, T=300)
        params = tuner_params(cfg)
        params["alpha0"] = np.linspace(0.0, 3.0, n)
        tb, params, st, traj, gap = _run(cfg, 300, params=params, record=list(range(n)))
        _check(cfg, tb, params, st, list(range(n)), 300, traj, arms=(n <= 3), gap=gap)


def test_step_replay_and_chunking_agree():
    """agft_step × T == one agft_replay(T) == chunked replays (resume from the workspace)."""
    cfg = _cfg("C2", n_tuners=4, n_traces=4, T=120)
    params = tuner_params(cfg)
    a = TunerBatch(cfg, params, device="cuda:0")
    rec = a.generate(0, 120)
    a.replay(rec, 0, 120)
    b = TunerBatch(cfg, params, device="cuda:0")
    for t0 in (0, 7, 64, 100):
        n = {0: 7, 7: 57, 64: 36, 100: 20}[t0]
        b.replay(b.generate(t0, n), t0, n)
    c = TunerBatch(cfg, params, device="cuda:0")
    chosen = []
    for t in range(120):
        chosen.append(c.step(c.generate(t, 1)).cpu().numpy())
    sa, sb, sc = a.stats(), b.stats(), c.stats()
    assert sa.tobytes() == sb.tobytes() == sc.tobytes()
    assert c.t == 120 and np.all(chosen[-1] == sa["last_arm"].astype(np.int32))
    for i in range(4):
        ea, eb = a.export_arms(i), b.export_arms(i)
        assert all(np.array_equal(ea[k], eb[k]) for k in ea)


def test_state_error_on_wrong_t0():
    cfg = _cfg("C1")
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    rec = tb.generate(0, 10)
    with pytest.raises(AgftError) as e:
        tb.replay(rec, 5, 10)
    assert e.value.code == -7
    tb.replay(rec, 0, 10)
    assert tb.t == 10


def test_invariants_on_gpu_state():
    """A⁻¹ symmetric (packed) and SPD with eigenvalues in (0, 1]; pruned arms never chosen."""
    cfg = _cfg("C2", n_tuners=8, n_traces=8)
    tb, params, st, traj, gap = _run(cfg, 1500, record=list(range(8)))
    for i in range(8):
        g = tb.export_arms(i)
        ev = np.linalg.eigvalsh(g["Ainv"])
        assert np.all(ev > 0) and np.all(ev <= 1 + 1e-12)
        assert g["active"][st["last_arm"][i]] == 1
        _, _, rec = oracle.run_tuner(cfg, oracle_tuner(params, i), T=1500, follow=traj[i], record=True)
        for t in range(1, 1500):
            m = rec["active_mask"][t - 1]
            k = int(traj[i][t])
            assert (m[k // 32] >> (k % 32)) & 1


def test_scheduled_kernels_agree_with_wide_at_scale():
    """All 4,096 C3 tuners: the class-scheduled kernels (WIDE → SEG → SOLO as arms are pruned)
    reproduce the one-warp-per-tuner schedule bit for bit wherever neither flagged a near-tie."""
    cfg = _cfg("C3")
    _, _, sa, _, _ = _run(cfg, 4500, policy=0)
    _, _, sw, _, _ = _run(cfg, 4500, policy=1)
    ok = (sa["near_tie_steps"] == 0) & (sw["near_tie_steps"] == 0)
    assert ok.mean() > 0.9
    assert np.array_equal(sa["traj_hash"][ok], sw["traj_hash"][ok])
    for f in ("sum_energy", "sum_edp", "sum_reward", "base_edp", "sum_active", "n_active"):
        assert np.array_equal(sa[f][ok], sw[f][ok]), f
    assert np.all(sa["steps"] == 4500) and np.all(sa["n_active"] >= 1)
    # the schedule really exercised the narrow classes
    assert (sa["n_active"] == 1).mean() > 0.5


def test_c5_rank_shard_sampled_parity():
    """C5 (1,048,576 tuners, 4,096 traces, pattern = trace mod 3) as rank 3 of an 8-GPU strong
    split: 131,072 local tuners on traces 1536…2047 (global Philox keys via trace_base), 3,000
    windows in the bench's launch configuration; sampled tuners against the oracle."""
    from paper_2508_01744_b200 import shard
    from _parity import compare_tuner
    cfg = _cfg("C5")
    sh = shard.plan(cfg, 8, 3, "strong")
    lcfg = dict(cfg, n_tuners=sh.n_tuners, n_traces=sh.n_traces)
    sample = [0, 1, 255, 256 * 100 + 77, 256 * 511 + 255]
    rec_slot = np.full(sh.n_tuners, NO_RECORD, np.uint32)
    for s, i in enumerate(sample):
        rec_slot[i] = s
    tb = TunerBatch(lcfg, sh.params, device="cuda:0", record_slot=rec_slot, trace_base=sh.trace_base)
    traj, _ = tb.run(3000, chunk=3000, record=True)
    st = tb.stats()
    assert np.all(st["steps"] == 3000) and np.all(st["flags"] == 0)
    problems = []
    for s, i in enumerate(sample):
        errs, _ = compare_tuner(lcfg, sh.params, i, st[i], tb.export_arms(i), 3000, traj[s],
                                trace_base=sh.trace_base)
        problems += errs
    assert not problems, "\n".join(problems[:20])
