import sys, numpy as np, torch, ctypes as C
sys.path.insert(0,'.')
from paper_1503_08294_b200 import _lib, workloads
lib=_lib.load_library(); ctx=_lib.default_context()
src, params, seed, desc = workloads.make("cfg3")
rng=np.random.Generator(np.random.Philox(3))
for n in (100, 500, 2000, 4000):
    pos = src.points[rng.integers(0, len(src.points), n)]
    sig = src.points[rng.integers(0, len(src.points), 4096)]
    out=[]
    for mode in (0, 2):
        dpos=torch.from_numpy(pos).cuda(); dsig=torch.from_numpy(sig).cuda()
        idx=torch.empty((4096,2),dtype=torch.int64,device='cuda'); d2=torch.empty((4096,2),dtype=torch.float64,device='cuda')
        _lib.check(lib.gs_find_device(ctx.handle, dpos.data_ptr(), n, dsig.data_ptr(), 4096, idx.data_ptr(), d2.data_ptr(), mode, None))
        torch.cuda.synchronize()
        fb=np.zeros(2,np.int64); _lib.check(lib.gs_find_last_fallback_counts(ctx.handle, fb))
        out.append((idx.cpu().numpy(), d2.cpu().numpy(), fb.copy()))
    print(n, "same:", np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1].view(np.int64), out[1][1].view(np.int64)), "fallbacks:", out[1][2])
