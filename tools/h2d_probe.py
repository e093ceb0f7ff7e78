import torch, time, numpy as np, sys
sys.path.insert(0, '.')
from paper_2105_04940_b200 import _lib
M = np.random.default_rng(0).standard_normal((500, 20000)); N = np.random.default_rng(1).standard_normal((20000, 500))
Mp, Np_ = torch.from_numpy(M).pin_memory(), torch.from_numpy(N).pin_memory()
Md, Nd = torch.empty(500*20000, dtype=torch.float64, device='cuda'), torch.empty(20000*500, dtype=torch.float64, device='cuda')
for it in range(5):
    torch.cuda.synchronize(); t=time.perf_counter()
    Md.copy_(Mp.view(-1), non_blocking=True); Nd.copy_(Np_.view(-1), non_blocking=True); torch.cuda.synchronize()
    t1=time.perf_counter()-t
    st=_lib.stream_ptr(); t=time.perf_counter()
    for c in range(8):
        c0, c1 = c*2500, (c+1)*2500
        _lib.call("bmm_copy2d", Md.data_ptr()+8*c0, 8*20000, Mp.data_ptr()+8*c0, 8*20000, 8*(c1-c0), 500, 1, st)
        nb = 8*(c1-c0)*500
        _lib.call("bmm_copy2d", Nd.data_ptr()+8*c0*500, nb, Np_.data_ptr()+8*c0*500, nb, nb, 1, 1, st)
    torch.cuda.synchronize(); t2=time.perf_counter()-t
    print(f"contiguous {t1*1e3:.2f} ms  chunked-2D {t2*1e3:.2f} ms")
