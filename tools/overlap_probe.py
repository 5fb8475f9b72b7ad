import sys, time, threading, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2502_12428_b200.engine import Engine
for p in (5, 7):
    c = bench.cached_block(p, 100000, 0, 0)
    dev = torch.from_numpy(c).cuda()
    for nctx in (1, 2, 3):
        engs = [Engine(p, 0) for _ in range(nctx)]
        for e in engs: e.set_workspace_limit(int(120e9 / nctx))
        parts = np.array_split(np.arange(100000), nctx)
        ins = [dev[int(ix[0]):int(ix[-1]) + 1].contiguous() for ix in parts]
        outs = [(torch.empty(len(ix), dtype=torch.int8, device="cuda"), torch.empty(len(ix), dtype=torch.int8, device="cuda")) for ix in parts]
        def work(k, reps):
            for _ in range(reps): engs[k].heights(ins[k], 10, out=outs[k])
        for k in range(nctx): work(k, 2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=work, args=(k, 6)) for k in range(nctx)]
        for t in th: t.start()
        for t in th: t.join()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 6
        print(f"p={p} contexts={nctx}: {dt*1e3:.2f} ms per 100k  ({1e5/dt/1e6:.2f} M/s)", flush=True)
        for e in engs: e.close()
