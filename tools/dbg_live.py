import sys; sys.path.insert(0, '.')
from dataclasses import replace
from paper_2602_16603_b200 import refsim
from paper_2602_16603_b200.config import SHAPES
from paper_2602_16603_b200.engine import synthetic_tokens
from paper_2602_16603_b200.live import run_live
from paper_2602_16603_b200.native import PrefillContext
ps = refsim.load()
shape = replace(SHAPES["llama3-8b"], num_layers=4)
ctx = PrefillContext(shape, kv_pages=256, max_pos=40000)
ctx.init_random(0)
reqs = [ps.Request(0, "file", 0.0, 16384, 10.0)]
for i in range(1, 6):
    reqs.append(ps.Request(i, "text", 0.004 * i, 300 + 50 * i, 0.05))
trace = ps.Trace(tuple(reqs))
res = run_live(trace, ps.PolicyConfig(), ps.CostParams(num_layers=4), ctx, synthetic_tokens(0, shape.vocab), record_events=True, max_wall_s=120)
for e in res.events: print(e)
