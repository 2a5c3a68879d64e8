"""GPU check of the Tables 2–5 reporting: the per-window series obtained by differencing the
CUDA replay's cumulative stats (report.windowed) equal the oracle's per-window record, and the
ablation runner produces the paper's three variants."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from agft_inputs import named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import TunerBatch, report  # noqa: E402

from _parity import oracle_tuner  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("bucket", [1, 75])
def test_windowed_series_match_the_oracle_record(bucket):
    T, n = 450, 3
    cfg = with_overrides(named_config("C2"), n_tuners=n, n_traces=n)
    params = tuner_params(cfg)
    tb = TunerBatch(cfg, params, device="cuda:0")
    s = report.windowed(tb, T, bucket)
    tb.close()
    for i in range(n):
        ost, _, rec = oracle.run_tuner(cfg, oracle_tuner(params, i), T=T, record=True)
        for k, rk in (("energy", "energy"), ("tpot", "tpot"), ("ttft", "ttft"), ("edp", "edp"),
                      ("reward", "reward")):
            want = rec[rk].reshape(-1, bucket).sum(axis=1) if bucket > 1 else rec[rk]
            np.testing.assert_allclose(s[k][:, i], want, rtol=1e-11, atol=1e-13, err_msg=k)
        assert s["base_energy"][:, i].sum() == pytest.approx(ost["base_energy"], rel=1e-12)
        assert int(s["final"]["traj_hash"][i]) == ost["traj_hash"]


def test_ablation_runner():
    T, n = 600, 2
    cfg = with_overrides(named_config("C2"), n_tuners=n, n_traces=n)
    ab = report.run_ablation(cfg, tuner_params(cfg), T, bucket=1)
    fin = {v: s["final"] for v, s in ab["series"].items()}
    assert np.all(fin["no_pruning"]["n_pruned_extreme"] + fin["no_pruning"]["n_pruned_hist"]
                  + fin["no_pruning"]["n_pruned_cascade"] == 0)
    assert np.all(fin["no_pruning"]["n_active"] == 107) and np.all(fin["no_grain"]["last_arm"] < 14)
    assert np.all(fin["full"]["n_active"] < 107)
    for v, t in ab["tables"].items():
        for m in ("energy", "edp", "tpot", "ttft"):
            assert np.isfinite(t[m]["mean"]) and np.isfinite(t[m]["cv"]), (v, m)
    tab = report.phase_tables(ab["series"]["full"], 231)
    assert tab["post"]["energy"]["diff_pct"] < 0            # AGFT saves energy against f_max
