"""Small invocations of every kernel of libagft.so, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): the class schedule (WIDE → SEG<32/16/8/4> → SOLO as pruning collapses the
action spaces), the WIDE schedule, the exploitation phase + refinement (both schedules), the ENV-C
closed loop, the offline sweep + regret, the live select / scores / observe step, and checkpoint /
attach.  Sizes are kept small: racecheck instruments every shared-memory access.
  compute-sanitizer --tool racecheck python tools/sanitize_driver.py [T]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from agft_inputs import live_inputs, named_config, tuner_params  # noqa: E402
from paper_2508_01744_b200 import TunerBatch  # noqa: E402


def main(T: int):
    c4 = dict(named_config("C4"), n_tuners=256, n_traces=1, T=T)          # one trace, all 256 sweep points
    cases = {
        "classes": (c4, 0),
        "wide": (c4, 1),
        "phase_classes": (dict(c4, ph_enable=1), 0),
        "refine_classes": (dict(c4, ph_enable=0, rf_enable=1), 0),
        "phase_refine_wide": (dict(c4, ph_enable=1, rf_enable=1), 0),
        "closed": (dict(c4, cl_enable=1), 0),
        "des": (dict(c4, cl_enable=2, n_tuners=64), 0),
        "C1": (named_config("C1"), 0),
    }
    for name, (cfg, pol) in cases.items():
        tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0", record_slot=[0] + [0xFFFFFFFF] * (cfg["n_tuners"] - 1),
                        policy=pol)
        tb.run(cfg["T"], chunk=max(1, cfg["T"] // 2), record=True)
        st = tb.stats()
        assert np.all(st["steps"] == cfg["T"]), name
        if name == "classes":
            if os.environ.get("SAN_NO_CHECKPOINT") != "1":   # initcheck: the checkpoint copies scratch regions
                ck = tb.checkpoint()
                tb2 = TunerBatch.resume(cfg, tuner_params(cfg), ck, device="cuda:0",
                                        record_slot=[0] + [0xFFFFFFFF] * (cfg["n_tuners"] - 1))
                tb2.close()
            sums = tb.new_sweep()
            tb.reset()
            rec = tb.generate(0, cfg["T"])
            tb.sweep(rec, 0, cfg["T"], sums, best=True)
            tb.regret(sums)
        torch.cuda.synchronize()
        tb.close()
        print(name, "ok", flush=True)
    c = dict(named_config("C2"), n_tuners=64, n_traces=64, sweep="none")
    rows, resp = live_inputs(dict(c, n_arms=1), 64, 40, seed=3)
    tb = TunerBatch(c, tuner_params(c), device="cuda:0")
    chosen = torch.empty(64, dtype=torch.int32, device="cuda:0")
    for t in range(40):
        r = torch.from_numpy(np.ascontiguousarray(rows[:, t]).view(np.int32)).cuda()
        tb.scores(r)
        tb.select(r, chosen)
        tb.observe(torch.from_numpy(np.ascontiguousarray(resp[:, t, 0])).cuda())
    torch.cuda.synchronize()
    tb.close()
    print("live ok", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 400)
