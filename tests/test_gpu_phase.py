"""GPU parity of the exploitation phase (ENV.md §4.10: Page-Hinkley detector, Eq. 2 greedy
selection) against the oracle, through the C-ABI, on every schedule that implements it."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from agft_inputs import named_config, tuner_params  # noqa: E402

from test_gpu_parity import _check, _run  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _cfg(name, **kw):
    c = named_config(name)
    c.update(ph_enable=1)
    c.update(kw)
    return c


@pytest.mark.parametrize("policy", [0, 1])
def test_c2_phase_parity(policy):
    cfg = _cfg("C2")
    tb, params, st, traj, gap = _run(cfg, 4500, record=[0], policy=policy)
    _check(cfg, tb, params, st, [0], 4500, traj, gap=gap)
    assert st["first_exploit_t"][0] != 0xFFFFFFFF and st["exploit_steps"][0] > 0


@pytest.mark.parametrize("kw", [
    dict(ph_window=1, ph_lambda=1e300),              # greedy (Eq. 2) from step 1 on
    dict(ph_window=5, ph_lambda=0.05),               # frequent alarms and re-entries
    dict(ph_window=20, ph_delta=0.0),
    dict(ph_window=3, hist_min_round=0, hist_min_samples=1),
    dict(ph_window=10, n_arms=33, f_step_mhz=45, prune_enable=0),
])
@pytest.mark.parametrize("policy", [0, 1])
def test_phase_edge_configs(kw, policy):
    cfg = _cfg("C2", n_tuners=5, n_traces=5, T=900)
    cfg.update(kw)
    ids = list(range(5))
    params = tuner_params(cfg, ids)
    params["alpha0"] = np.array([0.0, 0.3, 1.0, 2.0, 5.0])
    tb, params, st, traj, gap = _run(cfg, 900, params=params, record=ids, chunk=256, policy=policy)
    _check(cfg, tb, params, st, ids, 900, traj, gap=gap)


def test_c4_sweep_with_phase_sampled():
    """One C4 trace's 256 hyper-parameter points with the phase switch on, 20,000 windows, in
    the bench's launch configuration (all kernel classes, SOLO included)."""
    cfg = _cfg("C4", n_traces=1)
    ids = list(range(256))
    params = tuner_params(cfg, ids)
    sample = [0, 15, 48, 63, 100, 200, 255]
    tb, params, st, traj, gap = _run(cfg, 20000, params=params, record=sample, chunk=4500)
    _check(cfg, tb, params, st, sample, 20000, traj, gap=gap)
    assert np.all(st["steps"] == 20000) and np.all(st["flags"] == 0)
    assert (st["exploit_steps"] > 0).mean() > 0.5


# ------------------------------------------- ENV.md §4.11 refinement: WIDE (policy 1) and the class schedule
# with the deferred refinement pass at sub-chunk ends (policy 0 without the phase switch)
@pytest.mark.parametrize("kw", [
    dict(rf_enable=1),                                               # C2 defaults: statistical → predictive
    dict(rf_enable=1, ph_enable=1),                                  # + refinement on phase transitions
    dict(rf_enable=1, rf_period=7, rf_mature=300, rf_step_mhz=30),
    dict(rf_enable=1, ext_round_limit=200, ext_min_samples=1),       # many Extreme removals (permanent)
    dict(rf_enable=1, n_arms=35, f_step_mhz=45, rf_half_mhz=225, rf_step_mhz=45),
])
@pytest.mark.parametrize("policy", [0, 1])
def test_refinement_parity(kw, policy):
    cfg = named_config("C2")
    cfg.update(n_tuners=5, n_traces=5, T=1500, ph_enable=0)
    cfg.update(kw)
    ids = list(range(5))
    params = tuner_params(cfg, ids)
    params["alpha0"] = np.array([0.0, 0.3, 1.0, 2.0, 5.0])
    tb, params, st, traj, gap = _run(cfg, 1500, params=params, record=ids, chunk=512, policy=policy)
    _check(cfg, tb, params, st, ids, 1500, traj, gap=gap)
    assert np.all(st["n_refine"] > 0)


def test_refinement_c4_sample_class_schedule():
    """Refinement without the phase switch on the class schedule (deferred pass), C4 trace 0's
    256 tuners for 6,000 windows, a sample checked against the oracle."""
    cfg = named_config("C4")
    cfg.update(n_traces=1, rf_enable=1)
    ids = list(range(256))
    params = tuner_params(cfg, ids)
    sample = [0, 5, 31, 64, 130, 200, 255]
    tb, params, st, traj, gap = _run(cfg, 6000, params=params, record=sample, chunk=4500)
    _check(cfg, tb, params, st, sample, 6000, traj, gap=gap)


def test_refinement_c4_sample():
    cfg = named_config("C4")
    cfg.update(n_traces=1, rf_enable=1, ph_enable=1)
    ids = list(range(0, 256, 8))
    params = tuner_params(cfg, ids)
    tb, params, st, traj, gap = _run(cfg, 6000, params=params, record=list(range(len(ids))), chunk=4500)
    _check(cfg, tb, params, st, list(range(len(ids))), 6000, traj, gap=gap)
