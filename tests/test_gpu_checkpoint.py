"""Checkpoint / resume: a copy of the workspace plus the step counter, re-attached with
agft_attach, continues bit-identically — open loop, closed loop, phase switch + refinement."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2508_01744_b200 as pkg  # noqa: E402
from agft_inputs import named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import TunerBatch  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("kw", [{}, dict(cl_enable=1, pattern_mode=2), dict(ph_enable=1, rf_enable=1),
                                dict(rf_enable=1)])
def test_resume_is_bit_identical(kw):
    cfg = with_overrides(named_config("C2"), n_tuners=6, n_traces=6, **kw)
    params = tuner_params(cfg)
    a = TunerBatch(cfg, params, device="cuda:0")
    a.run(1700, chunk=600)
    state = a.checkpoint()
    assert state[1] == 1700
    a.run(3000, chunk=600)
    want = a.stats()
    b = TunerBatch.resume(cfg, params, state, device="cuda:0")
    assert b.t == 1700
    b.run(3000, chunk=600)
    got = b.stats()
    assert got.tobytes() == want.tobytes()
    for i in (0, 5):
        ea, eb = a.export_arms(i), b.export_arms(i)
        for f in ("Ainv", "b", "theta", "n", "rbar", "ebar", "active"):
            assert np.array_equal(ea[f], eb[f]), f
    a.close()
    b.close()


def test_attach_validates():
    cfg = with_overrides(named_config("C2"), n_tuners=2, n_traces=2)
    cfg_c = pkg.make_config(cfg)
    need = pkg.agft_workspace_bytes(cfg_c)
    small = torch.empty(need // 2, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(pkg.AgftError) as e:
        pkg.agft_attach(cfg_c, small, 0)
    assert e.value.code == -6
