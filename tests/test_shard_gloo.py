"""The N > 1 path on CPU: world_size-2 gloo process groups run the shard plan, the oracle on
each rank's shard, and the stats all-gather; the gathered result must equal one process
running every tuner (tuners never communicate)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from agft_inputs import named_config
from paper_2508_01744_b200 import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    c = named_config("C4")
    c.update(n_tuners=64, n_traces=4, T=120)          # 16 tuners per trace, tiny T
    return c


def _stats_array(stats_list):
    import oracle
    fields = oracle.STATS_FIELDS
    dt = np.dtype([(f, np.float64 if f.startswith(("sum_e", "sum_t", "sum_r", "base", "max")) else np.uint64)
                   for f in fields])
    return np.array([tuple(s[f] for f in fields) for s in stats_list], dtype=dt)


def _as_lib_stats(st):
    """The oracle's stats rows in the library's agft_tuner_stats layout (flags = 0: the oracle
    never freezes a tuner on these inputs), as shard.counter_vector reads them."""
    from paper_2508_01744_b200._abi import STATS_DTYPE
    out = np.zeros(len(st), dtype=STATS_DTYPE)
    for f in STATS_DTYPE.names:
        if f in st.dtype.names:
            out[f] = st[f]
    return out


def _worker(rank, world, port, scaling, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg()
    sh = shard.plan(cfg, world, rank, scaling)
    params = dict(sh.params)
    params["trace_id"] = params["trace_id"].astype(np.int64) + sh.trace_base   # oracle takes global ids
    st = _stats_array(oracle.run_batch(cfg, params, cfg["T"], threads=2))
    t = torch.from_numpy(st.view(np.uint8).copy())
    g = shard.gather_stats(t)
    mx = shard.max_over_ranks(float(rank + 1))
    cnt = shard.reduce_counters(shard.counter_vector(_as_lib_stats(st), cfg["T"]))
    if rank == 0:
        np.save(out_path, g.numpy())
        np.save(out_path + ".counters.npy", np.array([cnt[k] for k in shard.COUNTER_NAMES], dtype=np.int64))
        assert mx == float(world)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_rank_gloo_gather_matches_single_process(tmp_path, scaling):
    import oracle
    oracle.build()
    out = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(2, _free_port(), scaling, out), nprocs=2, join=True, start_method="spawn")
    gathered = np.load(out)
    cfg = _cfg()
    # single-process reference: all tuners of both shards in global order
    rows = []
    for r in range(2):
        sh = shard.plan(cfg, 2, r, scaling)
        p = dict(sh.params)
        p["trace_id"] = p["trace_id"].astype(np.int64) + sh.trace_base
        rows.append(_stats_array(oracle.run_batch(cfg, p, cfg["T"], threads=2)))
    ref = np.concatenate(rows)
    assert gathered.tobytes() == ref.view(np.uint8).tobytes()
    # the 16-counter all-reduce equals the counters of the single-process run
    counters = np.load(out + ".counters.npy")
    expect = shard.counter_vector(_as_lib_stats(ref), cfg["T"])
    assert counters.tolist() == expect
    assert expect[0] == cfg["n_tuners"] * (2 if scaling == "weak" else 1) * cfg["T"]


def test_plan_partitions():
    cfg = named_config("C5")
    seen = 0
    for r in range(8):
        sh = shard.plan(cfg, 8, r, "strong")
        assert sh.n_tuners == 131072 and sh.n_traces == 512 and sh.trace_base == 512 * r
        assert sh.params["trace_id"].max() < 512
        seen += sh.n_tuners
    assert seen == cfg["n_tuners"]
    c4 = named_config("C4")
    sh = shard.plan(c4, 4, 3, "weak")
    assert sh.n_tuners == 65536 and sh.trace_base == 3 * 256
    with pytest.raises(ValueError):
        shard.plan(dict(c4, n_tuners=65535), 2, 0, "strong")
