"""The CPU oracle under AddressSanitizer + UndefinedBehaviorSanitizer:
tests/sanitize/orc_san_driver.c links oracle/agft_oracle.c built with -fsanitize=address,undefined
(-fno-sanitize-recover: any finding aborts), runs every tuner with every per-step record and the final
arm state requested, re-runs it in follow mode along its own trajectory and sweeps trace 0.  The
sanitized build must be clean AND produce the same bytes as the production oracle build (the
floating-point flags of ENV.md §0 make the result independent of the optimisation level)."""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle
from agft_inputs import named_config, tuner_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "tests", "sanitize", "orc_san_driver.c")

pytestmark = pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc missing")


@pytest.fixture(scope="module")
def san_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("san") / "orc_san")
    subprocess.check_call(["gcc", "-std=c11", "-O1", "-g", "-ffp-contract=off", "-fno-fast-math",
                           "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer",
                           "-o", out, DRIVER, os.path.join(ROOT, "oracle", "agft_oracle.c"), "-lm", "-lpthread"])
    return out


def _cases():
    c1 = named_config("C1")
    c2 = dict(named_config("C2"), T=1500)
    c2p = dict(c2, ph_enable=1, rf_enable=1)
    c2c = dict(c2, cl_enable=1, T=900)
    c4 = dict(named_config("C4"), T=1200)
    aggressive = dict(c2, T=600, ext_round_limit=400, ext_min_samples=1, hist_min_round=5, hist_min_samples=2)
    return {"C1": (c1, [0]), "C2": (c2, [0]), "C2_phase_refine": (c2p, [0]), "C2_closed": (c2c, [0]),
            "C4_sweep_points": (c4, [0, 5, 17, 255]), "aggressive_pruning": (aggressive, [0])}


@pytest.mark.parametrize("name", list(_cases()))
def test_oracle_clean_under_asan_ubsan(san_bin, tmp_path, name):
    cfg, ids = _cases()[name]
    oc = oracle.make_config(cfg)
    p = tuner_params(cfg, ids)
    tuners = (oracle.OrcTuner * len(ids))(*[oracle.make_tuner(p["trace_id"][i], p["alpha0"][i],
                                                               p["ext_reward_threshold"][i], p["hist_k"][i])
                                            for i in range(len(ids))])
    fc, ft, fo = tmp_path / "cfg.bin", tmp_path / "tuners.bin", tmp_path / "out.bin"
    fc.write_bytes(bytes(oc))
    ft.write_bytes(bytes(tuners))
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([san_bin, str(fc), str(ft), str(cfg["T"]), str(fo)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "runtime error" not in r.stderr and "AddressSanitizer" not in r.stderr, r.stderr[-4000:]
    # the same bytes as the production build
    raw = fo.read_bytes()
    ns = C.sizeof(oracle.OrcStats)
    for i in range(len(ids)):
        st = oracle.OrcStats.from_buffer_copy(raw[i * ns:(i + 1) * ns])
        ref, _, _ = oracle.run_tuner(cfg, tuners[i], T=cfg["T"])
        for f in oracle.STATS_FIELDS:
            assert getattr(st, f) == ref[f], (name, i, f)
    K = cfg["n_arms"]
    off = len(ids) * ns
    acc, _ = oracle.sweep(cfg, 0, 0, cfg["T"])
    for key, dt, cnt in (("S", np.float64, K * 3), ("SP", np.float64, 5 * K), ("NP", np.uint32, 5),
                         ("O", np.float64, 2)):
        got = np.frombuffer(raw, dt, cnt, off)
        assert np.array_equal(got, np.asarray(acc[key]).reshape(-1)), key
        off += cnt * np.dtype(dt).itemsize
