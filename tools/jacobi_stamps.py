import ctypes, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2209_04876_b200 import _device as D, _lib
lib = _lib.load()
lib.ks_debug_jacobi_stamps.argtypes = [ctypes.c_void_p]
rng = np.random.default_rng(0)
for name, M in [("eye64", np.eye(64)), ("gram64", (lambda A: A.T @ A)(rng.normal(1, np.sqrt(1e-3), (16384, 64))))]:
    Mt = D.to_dev(M); s = D.empty(64); V = D.empty(64, 64)
    lib.ks_svd_small(D.p(Mt), 64, D.p(s), D.p(V), D.stream()); torch.cuda.synchronize()
    st = (ctypes.c_longlong * 4)(); lib.ks_debug_jacobi_stamps(st)
    lib.ks_svd_small(D.p(Mt), 64, D.p(s), D.p(V), D.stream()); torch.cuda.synchronize()
    lib.ks_debug_jacobi_stamps(st)
    r = max(st[3], 1)
    print(name, "rounds", st[3], "cycles/round: load+dot+shfl", st[0] / r, "rot+upd", st[1] / r, "barrier", st[2] / r)
