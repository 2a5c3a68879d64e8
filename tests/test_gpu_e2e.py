"""agft_run (the end-to-end C-ABI call: host params in, host stats out, trace generated in chunks
inside the call) against the handle-based path, open and closed loop, and the closed-loop
reporting series against the oracle's per-window record."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import paper_2508_01744_b200 as pkg  # noqa: E402
from agft_inputs import named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import TunerBatch, report  # noqa: E402

from _parity import oracle_tuner  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("kw", [{}, dict(cl_enable=1, pattern_mode=2)])
def test_agft_run_equals_the_handle_path(kw):
    T, chunk, n = 2000, 700, 8
    cfg = with_overrides(named_config("C2"), n_tuners=n, n_traces=n, **kw)
    params = tuner_params(cfg)
    tb = TunerBatch(cfg, params, device="cuda:0")
    tb.run(T, chunk=chunk)
    want = tb.stats()
    ws_bytes = tb.workspace.numel()
    tb.close()
    dev = torch.device("cuda:0")
    cfg_c = pkg.make_config(cfg, n_tuners=n, n_traces=n)
    hp = pkg.make_params(params)
    dp = torch.empty(hp.nbytes, dtype=torch.uint8, device=dev)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    per = pkg.RECORD_BYTES + (pkg.ROW_WORDS * 4 if kw.get("cl_enable") else 0)
    scratch = torch.empty(n * chunk * per, dtype=torch.uint8, device=dev)
    ds = torch.empty(n * pkg.STATS_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    hs = np.zeros(n, dtype=pkg.STATS_DTYPE)
    pkg.agft_run(cfg_c, hp, dp, T, chunk, ws, scratch, ds, hs)
    assert hs.tobytes() == want.tobytes()
    if kw.get("cl_enable"):                       # too small a scratch for the raw rows is refused
        small = torch.empty(n * chunk * pkg.RECORD_BYTES, dtype=torch.uint8, device=dev)
        with pytest.raises(pkg.AgftError) as e:
            pkg.agft_run(cfg_c, hp, dp, T, chunk, ws, small, ds, hs)
        assert e.value.code == -6


def test_closed_loop_report_series_match_the_oracle():
    T, n = 600, 2
    cfg = with_overrides(named_config("C2"), n_tuners=n, n_traces=n, cl_enable=1, pattern_mode=2)
    params = tuner_params(cfg)
    tb = TunerBatch(cfg, params, device="cuda:0")
    s = report.windowed(tb, T, bucket=1)
    tb.close()
    for i in range(n):
        ost, _, rec = oracle.run_tuner(cfg, oracle_tuner(params, i), T=T, record=True)
        for k in ("energy", "tpot", "ttft", "edp", "reward"):
            np.testing.assert_allclose(s[k][:, i], rec[k], rtol=1e-11, atol=1e-13, err_msg=k)
        assert int(s["final"]["traj_hash"][i]) == ost["traj_hash"]
        assert rec["backlog"].max() > 0            # the run did queue
