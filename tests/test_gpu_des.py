"""GPU parity of ENV-S, the discrete-event continuous-batching server (ENV.md §7; SPEC inference_sim
S:454-563), against the oracle: every tuner drives its own server at the
clocks it picks, each decision reads the server's last-window snapshot.  Trajectories, every stats
sum (energy, TPOT, TTFT, EDP, reward) and the arm state must match exactly as in the open-loop tests;
a checkpoint taken mid-run resumes bit-identically (the server state lives in the workspace)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from agft_inputs import named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import TunerBatch  # noqa: E402

from test_gpu_parity import _check, _run  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("kw,T,chunk", [
    (dict(pattern_mode=0), 1500, 700),                            # fluctuating prototypes
    (dict(pattern_mode=2), 1500, 4500),                           # bursts: queues and KV fill
    (dict(pattern_mode=2, kv_total=20000), 1200, 512),            # KV pressure: head-of-line waits
    (dict(pattern_mode=1, ph_enable=1, rf_enable=1), 1200, 1000),  # + phase switch + refinement
    (dict(pattern_mode=0, n_arms=1, prune_enable=0), 900, 300),    # one low clock: a saturated server
])
def test_des_parity(kw, T, chunk):
    cfg = with_overrides(named_config("C2"), cl_enable=2, n_tuners=6, n_traces=6, **kw)
    ids = list(range(6))
    params = tuner_params(cfg, ids)
    params["alpha0"] = np.array([0.0, 0.2, 0.5, 1.0, 2.0, 4.0])
    tb, params, st, traj, gap = _run(cfg, T, params=params, record=ids, chunk=chunk)
    _check(cfg, tb, params, st, ids, T, traj, gap=gap)
    assert np.all(st["steps"] == T) and np.all(st["flags"] == 0)
    assert np.all(st["base_energy"] == 0.0)                       # no f_max server under ENV-S
    tb.close()


def test_des_c4_trace_sampled():
    """One C4 trace's 256 hyper-parameter points on their own servers for 2,000 windows; a sample
    against the oracle."""
    cfg = with_overrides(named_config("C4"), cl_enable=2, n_traces=1)
    ids = list(range(256))
    params = tuner_params(cfg, ids)
    sample = [0, 15, 48, 63, 100, 200, 255]
    tb, params, st, traj, gap = _run(cfg, 2000, params=params, record=sample, chunk=1000)
    _check(cfg, tb, params, st, sample, 2000, traj, slots={i: s for s, i in enumerate(sample)}, gap=gap)
    tb.close()


def test_des_checkpoint_resume_bitidentical():
    cfg = with_overrides(named_config("C2"), cl_enable=2, n_tuners=4, n_traces=4, pattern_mode=2)
    params = tuner_params(cfg)
    ref = TunerBatch(cfg, params, device="cuda:0")
    ref.run(1000, chunk=250)
    want = ref.stats()
    tb = TunerBatch(cfg, params, device="cuda:0")
    tb.run(400, chunk=250)
    state = tb.checkpoint()
    tb.close()
    tb2 = TunerBatch.resume(cfg, params, state, device="cuda:0")
    tb2.run(1000, chunk=250)
    assert tb2.stats().tobytes() == want.tobytes()
    ref.close()
    tb2.close()


@pytest.mark.parametrize("kw", [
    dict(d=4),
    dict(median_window=1),
    dict(n_arms=1, prune_enable=0),
    dict(prune_enable=0),
    dict(kv_total=9000, pattern_mode=2),          # the queue overflows: arrivals are dropped
])
def test_des_edge_configs(kw):
    cfg = with_overrides(named_config("C2"), cl_enable=2, n_tuners=4, n_traces=4, **kw)
    ids = list(range(4))
    params = tuner_params(cfg, ids)
    tb, params, st, traj, gap = _run(cfg, 700, params=params, record=ids, chunk=350)
    _check(cfg, tb, params, st, ids, 700, traj, gap=gap)
    tb.close()
