"""Host-side profile of the live driver (paper_2602_16603_b200/live.py): wall time spent in the
reference scheduler (schedule_round), the reference timeline builder (build_timeline), task
creation and launch, per replay of the config-2 trace at a given rate -- the host work between a
completion and the next submit is GPU idle time in a single-slot execution pool.

    python tools/live_profile.py [--rate 85] [--duration 10] [--cost-params profiles/r1_bench_v15_relfit.log]
"""
import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_16603_b200 import live, refsim  # noqa: E402
from paper_2602_16603_b200.config import SHAPES  # noqa: E402
from paper_2602_16603_b200.native import PrefillContext, PrefillTask  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=85.0)
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--cost-params", default="profiles/r1_bench_v15_relfit.log")
    a = ap.parse_args()
    ps = refsim.load()
    line = open(a.cost_params).read().strip().splitlines()[-1]
    params = ps.CostParams.from_json_dict(json.loads(line)["goodput"]["cost_params"])
    shape = SHAPES[bench.MODEL]
    ctx = PrefillContext(shape, device=0, kv_pages=3000, page_size=128, max_pos=40000)
    ctx.init_random(seed=0)
    acc = collections.defaultdict(float)
    cnt = collections.Counter()

    def wrap(obj, name, key):
        f = getattr(obj, name)

        def g(*args, **kw):
            t0 = time.perf_counter()
            try:
                return f(*args, **kw)
            finally:
                acc[key] += time.perf_counter() - t0
                cnt[key] += 1
        setattr(obj, name, g)

    wrap(live, "schedule_round", "schedule_round")
    wrap(ps, "build_timeline", "build_timeline")
    wrap(PrefillContext, "create_task", "create_task")
    wrap(PrefillTask, "start", "task_start")
    wrap(PrefillTask, "poll", "task_poll")
    for rate in (a.rate,):
        for k in list(acc):
            acc[k] = 0.0
        cnt.clear()
        t0 = time.perf_counter()
        r = bench.live_run(ctx, shape, params, ps.PolicyConfig(), rate, a.duration)
        wall = time.perf_counter() - t0
        print(json.dumps({"rate": rate, "attainment": round(r["attainment"], 4), "wall_s": round(wall, 2),
                          "rounds": r["rounds"], "commands": r["commands"],
                          "host_s": {k: round(v, 3) for k, v in acc.items()},
                          "calls": dict(cnt)}))
    ctx.close()


if __name__ == "__main__":
    main()
