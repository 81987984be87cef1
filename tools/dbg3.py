import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, oracle_lib as O
from helpers import bits, canonical_perm
from paper_2202_06555_b200 import workloads as W
cfg = W.CONFIGS[3]; g = W.build_grid(cfg); keys, sur = g.nodes()
x = W.points(cfg, n=200)
nnz_o, h_o = O.port_grid_support(cfg.d, cfg.mode, keys, x); nnz, h = g.support(x)
bad = np.where(h != h_o)[0]
print("hash mismatch points", len(bad), bad[:10])
n = len(keys)
lv = np.floor(np.log2(keys.astype(np.float64))).astype(np.int64) + 1
ls = lv.sum(1)
run = np.zeros(n, int); r = 0
for i in range(1, n):
    a, b = keys[i-1], keys[i]
    asc = (ls[i-1] < ls[i]) or (ls[i-1] == ls[i] and tuple(a) < tuple(b))
    if not asc: r += 1
    run[i] = r
idx = ((keys - (1 << (lv-1))) * 2 + 1).astype(np.float64)
inv = np.ldexp(1.0, lv)
def fnv(seq):
    hh = 0xcbf29ce484222325
    for nn in seq:
        kk = int(nn)
        for byte in range(8):
            hh ^= (kk >> (8*byte)) & 0xff
            hh = (hh * 0x100000001b3) & 0xffffffffffffffff
    return hh
for p in bad[:3]:
    xx = x[p]
    t = xx[None,:] * inv
    v = np.where(lv == 1, 1.0, np.where(idx == 1, 2 - t, np.where(idx == inv - 1, 2 - (inv - t), 1 - np.abs(t - idx))))
    nz = np.where((v > 0).all(1))[0]
    rb = sorted(nz, key=lambda i: (run[i], ls[i], tuple(lv[i])))
    canon = sorted(nz, key=lambda i: (ls[i], tuple(lv[i])))
    print(p, "oracle", h_o[p], "gpu", h[p], "py-stored", fnv(nz), "py-run", fnv(rb), "py-canon", fnv(canon), "nnz", nnz[p], len(nz))
