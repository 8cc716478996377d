import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle import qc_oracle as O
from paper_2503_06545_b200 import device as D, _native as N
def t(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
def packed_from_codes(D, codes_kn, s, z, bits=8):
    K, Nn = codes_kn.shape
    buf = np.zeros((Nn, D.round16(K)), np.uint8); buf[:, :K] = codes_kn.T
    return D.PackedWeight(t(buf), t(np.asarray(s, np.float64)), t(np.asarray(z, np.int32)),
                          t(codes_kn.astype(np.int64).sum(0).astype(np.int32)), K, Nn, bits)
rng = np.random.default_rng(3)
S, K, Nn = 128, 256, 96
ca = rng.integers(0, 64, size=(S, K)).astype(np.uint8)
cw = rng.integers(0, 64, size=(K, Nn)).astype(np.uint8)
sw = O.scale_up16(rng.uniform(1e-3, 1e-2, size=Nn)); zw = rng.integers(0, 64, size=Nn).astype(np.int32)
a = D.ActCodes(t(np.pad(ca, ((0,0),(0,0)))), t(ca.astype(np.int64).sum(1).astype(np.int32)), t(np.array([2.0**-7])), t(np.array([3],np.int32)), K)
w = packed_from_codes(D, cw, sw, zw)
y = D.gemm_u8(a, w).cpu().numpy()
g = D.gemm_u8(a, w, epilogue=N.EPI_GELU).cpu().numpy()
want = O.gelu64(y)
bad = g != want
print("mismatch", bad.sum(), "of", g.size)
if bad.any():
    i = np.argwhere(bad)[:5]
    for r, c in i:
        print(y[r,c], g[r,c], want[r,c], np.frexp(want[r,c]), (g[r,c].view(np.int32)-want[r,c].view(np.int32)))
