import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2105_04940_b200 import _lib
torch.cuda.set_device(0)
lib, st = _lib.load(), _lib.stream_ptr()
bad = 0
for dt, B, r, c in [(torch.float64, 1, 500, 20000), (torch.float64, 3, 37, 200), (torch.float32, 2, 45, 100),
                    (torch.float64, 1, 1, 64), (torch.float32, 5, 333, 1000)]:
    g = torch.Generator().manual_seed(r * c)
    Xh = torch.randn((B, r, c), dtype=dt, generator=g)
    X = Xh.cuda()
    out = torch.zeros(B * c, dtype=torch.float64, device="cuda")
    lib.bmm_norms(_lib.matrix_dtype(X), X.data_ptr(), r, c, c, r * c, None, 0, 0, 0, B, 0, out.data_ptr(), None, st)
    torch.cuda.synchronize()
    x = Xh.numpy().astype(np.float64)
    ref = np.stack([np.add.reduce(x[b] * x[b], axis=0) for b in range(B)]).ravel()
    ok = np.array_equal(out.cpu().numpy(), ref)
    bad += not ok
    print(dt, B, r, c, "bit-exact" if ok else "MISMATCH")
sys.exit(bad)
