import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2502_12428_b200 as q
from paper_2502_12428_b200.engine import get_engine
for p, B in ((5, 100000), (7, 100000), (11, 4000), (11, 20000), (13, 2000)):
    c = torch.from_numpy(q.sample_block(p, B, 0, 0)).cuda()
    eng = get_engine(p, 0)
    for lazy in (False, True):
        for _ in range(3):
            h, i = eng.heights(c, 10, lazy=lazy)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            h, i = eng.heights(c, 10, lazy=lazy)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        st = eng.stats()
        print(p, B, "lazy" if lazy else "eager", f"{dt*1e3:.3f} ms/step {B/dt/1e6:.3f} M/s", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items() if k.startswith("ms_") or k in ("hard", "built", "chunks")}, flush=True)
