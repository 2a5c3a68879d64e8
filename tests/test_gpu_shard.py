"""The library's N > 1 path on one GPU: two gloo ranks share cuda:0, each runs
its strong-scaling shard of a C4-shaped sweep through the C-ABI library (its own traces, no input
exchange), the per-tuner stats are all-gathered and the 16 run counters all-reduced.  Tuners never
communicate, so the gathered bytes must equal one process replaying every tuner, and the
all-reduced counters must equal that process's counters."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from agft_inputs import named_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    c = named_config("C4")
    c.update(n_tuners=512, n_traces=8, T=3000)       # 64 tuners per trace: α × pruning points 0..63
    return c


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2508_01744_b200 import TunerBatch, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = _cfg()
    sh = shard.plan(cfg, world, rank, "strong")
    tb = TunerBatch(dict(cfg, n_tuners=sh.n_tuners, n_traces=sh.n_traces), sh.params, device="cuda:0",
                    trace_base=sh.trace_base)
    tb.run(cfg["T"], chunk=1000)
    st = tb.stats_tensor().cpu()
    g = shard.gather_stats(st)
    cnt = shard.reduce_counters(shard.counter_vector(st.numpy().view(tb_dtype()), cfg["T"]))
    if rank == 0:
        np.save(out_path, g.numpy())
        np.save(out_path + ".counters.npy", np.array([cnt[k] for k in shard.COUNTER_NAMES], dtype=np.int64))
    dist.barrier()
    tb.close()
    dist.destroy_process_group()


def tb_dtype():
    from paper_2508_01744_b200 import STATS_DTYPE
    return STATS_DTYPE


def test_two_gloo_ranks_on_one_gpu_match_single_process(tmp_path):
    from paper_2508_01744_b200 import TunerBatch, shard, STATS_DTYPE
    from agft_inputs import tuner_params
    out = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    gathered = np.load(out)
    cfg = _cfg()
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    tb.run(cfg["T"], chunk=1500)                        # different chunking: the result must not depend on it
    st = tb.stats()
    assert gathered.tobytes() == st.view(np.uint8).tobytes()
    counters = np.load(out + ".counters.npy").tolist()
    assert counters == shard.counter_vector(st, cfg["T"])
    assert counters[0] == cfg["n_tuners"] * cfg["T"] and counters[1] == 0 and counters[3] == 0
    tb.close()
