import sys; sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2601_07508_b200 as F
import oracle as O
for eng in (F.ENGINE_RNS, F.ENGINE_I8, F.ENGINE_DMMA):
    m = k = n = 1024; bits = 50
    p = F.prev_prime(1 << bits)
    pl = F.plan_for_modulus(p, m, k, n)
    A = torch.empty((m, k), dtype=torch.float64, device='cuda'); B = torch.empty((k, n), dtype=torch.float64, device='cuda')
    C = torch.empty((m, n), dtype=torch.float64, device='cuda')
    F.random_residues_device(A, p, 1); F.random_residues_device(B, p, 2)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, stream=s, flags=eng | F.ASYNC)  # warm-up: workspaces
    torch.cuda.synchronize()
    ref = C.clone()
    g = torch.cuda.CUDAGraph()
    C.zero_()
    with torch.cuda.graph(g, stream=s):
        F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, stream=s, flags=eng | F.ASYNC)
    C.zero_(); torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    print(eng, 'graph replay equal:', torch.equal(C, ref))
    # timing: graph replay vs direct
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(20): g.replay()
    e1.record(); torch.cuda.synchronize(); tg = e0.elapsed_time(e1)/20
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(20): F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, stream=s, flags=eng | F.ASYNC)
    e1.record(s); torch.cuda.synchronize(); td = e0.elapsed_time(e1)/20
    print(eng, 'graph %.3f ms, direct %.3f ms' % (tg, td))
