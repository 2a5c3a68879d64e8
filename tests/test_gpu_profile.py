"""The measurement API (agft_profile_start / agft_profile_read, agft_occupancy): the per-class
tuner-step counters of a replay add up to every tuner's steps, Σ K_act to the stats' sum_active, in
both the concurrent and the serialised mode, and every class has a positive residency."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2508_01744_b200 as pkg  # noqa: E402
from agft_inputs import named_config, tuner_params  # noqa: E402
from paper_2508_01744_b200 import TunerBatch, make_config  # noqa: E402
from paper_2508_01744_b200._abi import PROFILE_SLOTS  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("serialize", [False, True])
def test_profile_counters_add_up(serialize):
    cfg = dict(named_config("C4"), n_tuners=512, n_traces=2, T=3000)
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    pkg.agft_profile_start(tb.h, serialize)
    tb.run(cfg["T"], chunk=1500)
    prof = pkg.agft_profile_read(tb.h)
    st = tb.stats()
    steps = sum(v["tuner_steps"] for v in prof.values())
    act = sum(v["active_arm_steps"] for v in prof.values())
    assert steps == 512 * cfg["T"] == int(st["steps"].astype(np.int64).sum())
    assert act == int(st["sum_active"].astype(np.int64).sum())
    assert prof["classify"]["launches"] > 0 and all(v["kernel_ms"] >= 0 for v in prof.values())
    used = [k for k, v in prof.items() if v["tuner_steps"] > 0]
    assert "solo" in used and any(k.startswith("seg") for k in used)
    tb.close()


def test_occupancy_is_positive_for_every_class():
    c = make_config(dict(named_config("C2"), n_tuners=1, n_traces=1), n_tuners=1, n_traces=1)
    for slot, name in enumerate(PROFILE_SLOTS[:6]):
        assert pkg.agft_occupancy(c, slot) > 0, name
