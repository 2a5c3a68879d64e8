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


def test_checkpoint_carries_sweep_counter_and_refuses_pending_select():
    """the sweep counter is part of the checkpoint; a checkpoint between agft_select and
    agft_observe is refused (the pending selection is not workspace state)."""
    from agft_inputs import live_inputs
    cfg = with_overrides(named_config("C2"), n_tuners=2, n_traces=2)
    params = tuner_params(cfg)
    a = TunerBatch(cfg, params, device="cuda:0")
    rec = a.generate(0, 300)
    sums = a.new_sweep()
    a.sweep(rec, 0, 300, sums)
    a.replay(rec, 0, 300)
    state = a.checkpoint()
    assert state[1] == 300 and state[2] == 300
    b = TunerBatch.resume(cfg, params, state, device="cuda:0")
    rec2 = b.generate(300, 100)
    b.sweep(rec2, 300, 100, sums)                     # continues the chunked sweep (t0 == sweep_t)
    rows, _ = live_inputs(cfg, 2, 1, seed=3)
    b.select(torch.from_numpy(np.ascontiguousarray(rows[:, 0]).view(np.int32)).to("cuda:0"))
    with pytest.raises(pkg.AgftError) as e:
        b.checkpoint()
    assert e.value.code == -7
    a.close()
    b.close()


def test_create_rejects_out_of_range_params():
    """trace_id ≥ n_traces, a record_slot outside [0, record_slots) that is not
    NO_RECORD, or a non-finite α0 are rejected at agft_create (AGFT_E_INVALID_ARG)."""
    cfg = with_overrides(named_config("C2"), n_tuners=4, n_traces=2)
    for bad in ({"trace_id": 2}, {"alpha0": float("nan")}, {"alpha0": -1.0}, {"hist_k": float("inf")}):
        params = tuner_params(cfg)
        params["trace_id"] = np.array(params["trace_id"]) % 2
        for k, v in bad.items():
            arr = np.array(params[k], dtype=np.float64 if k != "trace_id" else np.uint32)
            arr[1] = v
            params[k] = arr
        with pytest.raises(pkg.AgftError) as e:
            TunerBatch(cfg, params, device="cuda:0")
        assert e.value.code == -1, bad
    params = tuner_params(cfg)
    params["trace_id"] = np.array(params["trace_id"]) % 2
    cfg_c = pkg.make_config(cfg, record_slots=2)       # 2 record rows, tuner 1 asks for row 5
    host = pkg.make_params(params, np.array([0, 5, pkg.NO_RECORD, pkg.NO_RECORD], dtype=np.uint32))
    d_params = torch.from_numpy(host.view(np.uint8)).to("cuda:0")
    ws = torch.empty(pkg.agft_workspace_bytes(cfg_c), dtype=torch.uint8, device="cuda:0")
    with pytest.raises(pkg.AgftError) as e:
        pkg.agft_create(cfg_c, d_params, ws)
    assert e.value.code == -1


def test_frozen_tuner_reads_never_in_step_output():
    """a tuner frozen by a non-finite measurement is not scheduled; agft_step reports
    AGFT_NEVER (-1 as int32) for it instead of an uninitialised value."""
    from agft_inputs import live_inputs
    cfg = with_overrides(named_config("C2"), n_tuners=3, n_traces=3)
    params = tuner_params(cfg)
    tb = TunerBatch(cfg, params, device="cuda:0")
    rows, resp = live_inputs(cfg, 3, 1, seed=5)
    k = tb.select(torch.from_numpy(np.ascontiguousarray(rows[:, 0]).view(np.int32)).to("cuda:0")).cpu().numpy()
    m = np.ascontiguousarray(resp[np.arange(3), 0, k]).copy()
    m[1, 0] = float("nan")
    tb.observe(torch.from_numpy(m).to("cuda:0"))
    assert int(tb.stats()["flags"][1]) & 1
    rec = tb.generate(1, 1)
    ch = tb.step(rec).cpu().numpy()
    assert ch[1] == -1 and ch[0] >= 0 and ch[2] >= 0
    tb.close()


def test_regret_refused_on_closed_loop_handle():
    """the offline sweep is open-loop (ENV.md §5); per-tuner regret against it is
    meaningless for a closed-loop handle."""
    cfg = with_overrides(named_config("C2"), n_tuners=2, n_traces=2, cl_enable=1)
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    rec = tb.generate(0, 50)
    sums = tb.new_sweep()
    tb.sweep(rec, 0, 50, sums)
    with pytest.raises(pkg.AgftError) as e:
        tb.regret(sums)
    assert e.value.code == -1
    tb.close()
