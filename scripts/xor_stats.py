"""XOR-key aligned layout statistics of the TFIM-10 Liouvillian (oracle L): per 32-row slice, the
union of keys col^row (slice width), against the SELL width (max row length); distinct values
per warp instruction in both layouts."""
import numpy as np, sys
sys.path.insert(0, '/root/repo')
from oracle import oracle as O
m = O.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
rp, col, val, n = m.export(O.L_CONST)
rp = np.asarray(rp); col = np.asarray(col).astype(np.int64)
val = np.asarray(val)
val = val.view(np.complex128) if val.dtype != np.complex128 else val
lens = np.diff(rp); rows = np.repeat(np.arange(n), lens)
key = col ^ rows
vu, vc = np.unique(np.stack([val.real.view(np.int64), val.imag.view(np.int64)], 1), axis=0, return_inverse=True)
vc = vc.ravel()
print("nnz", len(col), "distinct values", len(vu), "distinct keys", len(np.unique(key)))
nsl = n // 32
sl = rows // 32
# union width per slice
pair = np.unique(sl * (1 << 40) + key)
ws = np.bincount(pair >> 40, minlength=nsl)
wsell = lens.reshape(nsl, 32).max(1)
print("xor width: mean %.2f max %d | sell width mean %.2f; xor code slots %d vs sell %d" %
      (ws.mean(), ws.max(), wsell.mean(), 32 * ws.sum(), 32 * ((wsell + 7) // 8 * 8).sum()))
# distinct values per instruction (slice, position) in the xor layout
samp = np.arange(0, nsl, 97)
tv = cnt = 0
for s in samp:
    msk = sl == s
    k = key[msk]; v = vc[msk]
    uk = np.unique(k)
    for kk in uk:
        tv += len(np.unique(v[k == kk])); cnt += 1
print("xor layout: distinct values / instr %.2f" % (tv / cnt))
