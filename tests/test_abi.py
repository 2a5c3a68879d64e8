"""CPU-side checks of the C-ABI boundary: the library builds and loads, exports every
entry point include/agft.h declares, its struct mirrors match, and host validation
returns the documented status codes. No kernel is launched here."""
import math

import numpy as np
import os
import re

import pytest

import paper_2508_01744_b200 as pkg
from paper_2508_01744_b200 import _abi
from agft_inputs import named_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "agft.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2508_01744_b200 import build
    build.build()
    return _abi.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(agft_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("agft_create", "agft_step", "agft_replay", "agft_stats"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
        assert n in _abi.PROTOTYPES, f"binding lacks {n}"


def test_struct_mirrors_match(lib):
    assert lib.agft_struct_size(0) == __import__("ctypes").sizeof(_abi.AgftConfig)
    assert lib.agft_struct_size(1) == 32
    assert lib.agft_struct_size(2) == 128


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_named_configs_validate(lib, name):
    c = _abi.make_config(named_config(name))
    assert lib.agft_validate(c) == 0
    assert pkg.agft_workspace_bytes(c) > 0


def _bad(lib, **kw):
    cfg = named_config("C2")
    cfg.update(kw)
    return lib.agft_validate(_abi.make_config(cfg))


def test_validation_codes(lib):
    assert _bad(lib, n_arms=0) == -3                         # S:161 empty arm set
    assert _bad(lib, f_step_mhz=0) == -2                     # S:271 invalid grid
    assert _bad(lib, n_arms=129) == -2
    assert _bad(lib, n_arms=108) == -2                       # 210 + 107·15 > 1800
    assert _bad(lib, d=0) == -4 and _bad(lib, d=8) == -4
    assert _bad(lib, tau=math.nan) == -5                     # S:181 non-finite
    assert _bad(lib, p_idle=-1.0) == -5
    assert _bad(lib, u_max=1.0) == -5
    assert _bad(lib, median_window=0) == -1 and _bad(lib, median_window=65) == -1
    assert _bad(lib, weight=[1, 2, 3, 4, 5]) == -1
    assert _bad(lib, norm_lo=[2.0] * 7) == -5                # lo > hi
    c = _abi.make_config(named_config("C2"))
    c.abi_version = 99
    assert lib.agft_validate(c) == -1
    c.abi_version = _abi.ABI_VERSION
    c.n_tuners = 0
    assert pkg.agft_workspace_bytes(c) == 0


def test_workspace_scales_with_tuners(lib):
    w1 = pkg.agft_workspace_bytes(_abi.make_config(named_config("C2"), n_tuners=1024, n_traces=1))
    w2 = pkg.agft_workspace_bytes(_abi.make_config(named_config("C2"), n_tuners=2048, n_traces=1))
    assert w1 > 0 and w2 > w1
    # ≈ 46 KB of canonical tuner state per tuner (K padded to 128 arms, d = 7)
    assert 40_000 < (w2 - w1) / 1024 < 50_000


def test_status_strings(lib):
    for code, text in _abi.STATUS.items():
        assert lib.agft_status_string(code).decode() == text


def test_create_without_device_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import ctypes
    import numpy as np
    c = _abi.make_config(named_config("C1"))
    buf = np.zeros(pkg.agft_workspace_bytes(c) + 256, np.uint8)
    base = (buf.ctypes.data + 255) // 256 * 256
    h = ctypes.c_void_p()
    params = np.zeros(1, _abi.PARAMS_DTYPE)
    rc = lib.agft_create(ctypes.byref(c), params.ctypes.data, base, buf.nbytes - 256, None, ctypes.byref(h))
    assert rc in (-9, -8)


def test_product_never_imports_the_oracle():
    pdir = os.path.join(ROOT, "paper_2508_01744_b200")
    for dirpath, _, files in os.walk(pdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\b(import|from)\s+oracle\b", txt), f
                assert "agft_oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"\b(import|from)\s+paper_2508_01744_b200\b", txt), f
            assert not re.search(r'#include\s+"[^"]*(agft\.h|agft_internal)', txt), f


def test_record_slot_count():
    """Rows of the trajectory record for partially recorded batches (uint32 NO_RECORD markers)."""
    import numpy as np
    r = np.full(10, pkg.NO_RECORD, np.uint32)
    assert pkg.record_slot_count(r) == 0 and pkg.record_slot_count(None) == 0
    r[3], r[7] = 0, 4
    assert pkg.record_slot_count(r) == 5
    assert pkg.record_slot_count(np.arange(6, dtype=np.uint32)) == 6


def test_closed_loop_and_attach_host_checks(lib):
    """ABI v5/v8: agft_closed validation (1 ENV-C, 2 ENV-S, nothing else), the ENV-S workspace, and
    agft_attach's host-side checks (no kernel launched)."""
    import ctypes
    import numpy as np
    assert _bad(lib, cl_enable=3) == -1
    assert _bad(lib, cl_enable=2) == 0
    c1 = _abi.make_config(dict(named_config("C2"), n_tuners=10), n_tuners=10)
    c2 = _abi.make_config(dict(named_config("C2"), n_tuners=10, cl_enable=2), n_tuners=10)
    # ENV-S adds the server of every tuner: 128-B scalars + 512 queued + 128 running requests of 24 B
    assert pkg.agft_workspace_bytes(c2) - pkg.agft_workspace_bytes(c1) >= 10 * (128 + 640 * 24)
    assert _bad(lib, cl_enable=1, cl_q_max=0) == 0            # a zero cap is the open loop (ENV.md §6)
    c = _abi.make_config(named_config("C2"))
    h = ctypes.c_void_p()
    need = pkg.agft_workspace_bytes(c)
    buf = np.zeros(need + 512, np.uint8)
    base = (buf.ctypes.data + 255) // 256 * 256
    assert lib.agft_attach(ctypes.byref(c), base, need - 1, None, 0, 0, ctypes.byref(h)) == -6
    assert lib.agft_attach(ctypes.byref(c), base + 8, need, None, 0, 0, ctypes.byref(h)) == -6   # misaligned
    c.abi_version = 99
    assert lib.agft_attach(ctypes.byref(c), base, need, None, 0, 0, ctypes.byref(h)) == -1
    assert not h.value


def test_bench_parity_summary_counts():
    """bench.py's in-line parity check: hashes first, then every exact field, on any sample size."""
    import numpy as np
    import bench
    g = np.zeros(3, dtype=_abi.STATS_DTYPE)
    g["traj_hash"] = [1, 2, 3]
    g["sum_edp"] = [1.0, 2.0, 3.0]
    ost = [{f: 0 for f in bench.PARITY_EXACT} for _ in range(2)]
    for i, o in enumerate(ost):
        o["traj_hash"] = int(g["traj_hash"][i])
        o["sum_edp"] = float(g["sum_edp"][i])
    ost[1]["sum_edp"] = 2.5                                    # same path, different sum
    p = bench.parity_summary(g, ost)
    assert p["tuners"] == 2 and p["traj_hash_match"] == 2 and p["stats_exact_given_traj"] == 1


def test_agft_run_validates_host_params_before_touching_the_device(lib):
    """agft_run rejects a trace_id ≥ n_traces (or a non-finite α0) in the HOST params
    with AGFT_E_INVALID_ARG before any copy or launch — so this runs without a GPU."""
    import ctypes as C
    from agft_inputs import tuner_params
    cfg = dict(named_config("C2"), n_tuners=4, n_traces=2)
    cfg_c = _abi.make_config(cfg)
    params = tuner_params(cfg)
    for field, val in (("trace_id", 7), ("alpha0", float("nan"))):
        p = dict(params)
        arr = np.array(p[field if field != "alpha0" else "alpha0"], dtype=np.float64 if field == "alpha0" else np.uint32)
        arr[2] = val
        p[field] = arr
        if field != "trace_id":
            p["trace_id"] = np.array(params["trace_id"]) % 2
        hp = _abi.make_params(p)
        dummy = np.zeros(64, np.uint8)
        code = lib.agft_run(C.byref(cfg_c), hp.ctypes.data, dummy.ctypes.data, 10, 10, dummy.ctypes.data, 1 << 40,
                            dummy.ctypes.data, 1 << 40, dummy.ctypes.data, dummy.ctypes.data, None)
        assert code == -1, field
