import sys, numpy as np
sys.path.insert(0, '.')
from oracle import forward as F
from paper_2602_16603_b200.config import SHAPES
from paper_2602_16603_b200.native import PrefillContext
shape = F.SHAPES["tiny-moe"]; w = F.make_weights(shape, 1234)
ctx = PrefillContext(SHAPES["tiny-moe"], kv_pages=512, page_size=128, max_pos=8192); ctx.load_weights(w)
def rel(a,b): return float(np.abs(a-b).max()/max(np.abs(b).max(),1e-6))
for lens, chunk in [([1000,5],256), ([1000,5],None), ([1000],256), ([600],None), ([600],300)]:
    toks = F.make_tokens(lens, shape.vocab, 77)
    ot = F.OracleTask(shape, w, toks, chunk); ot.run_all()
    t = ctx.create_task(toks, chunk, "operator"); t.begin_segment(0); t.enqueue(0, t.n_entries); ctx.sync()
    print(lens, chunk, "logits", rel(t.logits(), ot.logits))
    for r in range(len(lens)):
        for layer in range(shape.num_layers):
            k, v = t.read_kv(r, layer)
            kr = ot.k_cache[r][layer]
            rowerr = np.abs(k - kr).max(axis=(1,2)) / np.abs(kr).max()
            bad = np.nonzero(rowerr > 0.03)[0]
            print(f"  r={r} L={layer} kerr={rel(k,kr):.4f} verr={rel(v, ot.v_cache[r][layer]):.4f} bad_rows={bad[:10]} n_bad={len(bad)}")
    t.destroy()
ctx.close()
