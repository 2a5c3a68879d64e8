"""Host logic of the Tables 2–5 reporting (paper_2508_01744_b200/report.py): bucketing and
differencing of cumulative stats, means, CVs, the pre/post split and the ablation configs.
CPU only: a fake batch stands in for the CUDA replay."""
import numpy as np
import pytest

from agft_inputs import named_config
from paper_2508_01744_b200 import _abi, report
from paper_2508_01744_b200._abi import STATS_DTYPE


class FakeBatch:
    """Cumulative stats of N tuners whose window t contributes E = 1 + t + i, TPOT = 0.01·(i+1)."""

    def __init__(self, n):
        self.n, self.t = n, 0
        self.st = np.zeros(n, dtype=STATS_DTYPE)
        self.calls = []

    def stats(self):
        return self.st.copy()

    def new_records(self, m):
        return np.zeros((1, m))

    def generate(self, t, m, rec):
        assert t == self.t

    def replay(self, rec, t, m):
        self.calls.append((t, m))
        for s in range(t, t + m):
            for i in range(self.n):
                E, tp = 1.0 + s + i, 0.01 * (i + 1)
                self.st["sum_energy"][i] += E
                self.st["sum_tpot"][i] += tp
                self.st["sum_edp"][i] += E * tp
                self.st["base_energy"][i] += 2.0 * E
                self.st["base_edp"][i] += 2.0 * E * 0.5 * tp
                self.st["steps"][i] += 1
        self.t += m


def test_windowed_buckets_and_ragged_tail():
    fb = FakeBatch(3)
    s = report.windowed(fb, 10, bucket=4)
    assert fb.calls == [(0, 4), (4, 4), (8, 2)]
    assert list(s["t0"]) == [0, 4, 8]
    assert s["steps"][:, 0].tolist() == [4, 4, 2]
    assert s["energy"][2, 1] == (1 + 8 + 1) + (1 + 9 + 1)
    w = report.per_window(s)
    np.testing.assert_allclose(w["energy"][:, 0], [2.5, 6.5, 9.5])
    np.testing.assert_allclose(w["base_tpot"][:, 2], 0.015)          # base EDP / base E


def test_mean_cv_definition():
    x = np.array([[1.0, 2.0], [3.0, 2.0]])          # tuner 0: mean 2, std 1; tuner 1: constant
    mu, cv = report.mean_cv(x)
    assert mu == 2.0 and cv == 0.25


def test_phase_tables_split():
    fb = FakeBatch(2)
    s = report.windowed(fb, 6, bucket=1)
    tab = report.phase_tables(s, 2)
    assert tab["pre"]["windows"] == 4 and tab["post"]["windows"] == 8
    e_pre = np.mean([1 + t + i for t in (0, 1) for i in (0, 1)])
    assert tab["pre"]["energy"]["agft"] == pytest.approx(e_pre)
    assert tab["pre"]["energy"]["diff_pct"] == pytest.approx(-50.0)    # base E = 2 E
    assert tab["post"]["tpot"]["diff_pct"] == pytest.approx(100.0)     # base TPOT = TPOT / 2
    per = np.array([1, 5])                                            # per-tuner split
    assert report.phase_tables(s, per)["pre"]["windows"] == 6


def test_ablation_configs_validate():
    cfg = named_config("C2")
    ab = report.ablation_configs(cfg)
    ng = ab["no_grain"]
    assert ng["n_arms"] == 14 and ng["f_step_mhz"] == 120
    assert ng["f_min_mhz"] + (ng["n_arms"] - 1) * ng["f_step_mhz"] == 1770
    assert ab["no_pruning"]["prune_enable"] == 0 and ab["full"] == cfg
    lib = _abi.lib()
    for c in ab.values():
        assert lib.agft_validate(_abi.make_config(c)) == 0


def test_cv_table_diffs():
    a, b = FakeBatch(2), FakeBatch(2)
    sa, sb = report.windowed(a, 5), report.windowed(b, 5)
    sb = {k: (v * 2.0 if k in ("energy", "edp") else v) for k, v in sb.items()}
    t = report.cv_table({"full": sa, "no_grain": sb})
    assert t["no_grain"]["energy"]["mean_diff_pct"] == pytest.approx(100.0)
    assert t["no_grain"]["energy"]["cv_diff_pct"] == pytest.approx(0.0, abs=1e-9)
