"""Failure detection (A⁻¹ stays symmetric positive definite, eigenvalues in
(0, 1] since λ_min(A) ≥ 1).  A tuner whose arm state is corrupted — here the diagonal of every arm's
A⁻¹ overwritten with −1 in a checkpointed workspace — must be frozen after its next update with
stats.flags bit 0 (frozen) and bit 1 (SPD violation) set, on every kernel class (WIDE, SEG, SOLO),
while the other tuners of the batch continue bit-identically to an uncorrupted resume."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from agft_inputs import named_config, tuner_params  # noqa: E402
from paper_2508_01744_b200 import TunerBatch  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("policy,pre", [(1, 200), (0, 200), (0, 3000)])   # WIDE; classes early / late (SEG, SOLO)
def test_spd_violation_freezes_only_that_tuner(policy, pre):
    cfg = dict(named_config("C2"), n_tuners=6, n_traces=6)
    params = tuner_params(cfg)
    T = pre + 400
    tb = TunerBatch(cfg, params, device="cuda:0", policy=policy)
    tb.run(pre, chunk=pre)
    ws, t, sw = tb.checkpoint()
    tb.close()
    ref = TunerBatch.resume(cfg, params, (ws.clone(), t, sw), device="cuda:0", policy=policy)
    ref.run(T, chunk=200)
    want = ref.stats()
    ref.close()
    # corrupt tuner 3: every arm's A⁻¹ diagonal (the workspace starts with A⁻¹ [N][P][128], ENV layout)
    d = cfg["d"]
    P = d * (d + 1) // 2
    a = ws.numpy().view(np.float64)
    bad = 3
    for r in range(d):
        e = r * d - r * (r - 1) // 2
        a[(bad * P + e) * 128:(bad * P + e) * 128 + cfg["n_arms"]] = -1.0
    tb2 = TunerBatch.resume(cfg, params, (ws, t, sw), device="cuda:0", policy=policy)
    tb2.run(T, chunk=200)
    got = tb2.stats()
    tb2.close()
    assert got["flags"][bad] & 3 == 3
    assert pre <= got["steps"][bad] <= pre + 1            # frozen at its first update after the resume
    for i in range(cfg["n_tuners"]):
        if i != bad:
            assert got[i].tobytes() == want[i].tobytes()
    assert np.all(want["flags"] == 0)
