"""Key-aligned store statistics: per 32-row slice, the sorted union of keys
col ^ row; per (slice, key) position, whether every present lane carries the same value
(warp-uniform) or not (per-lane value ids). Prints the store size the layout would take."""
import sys

import numpy as np

sys.path.insert(0, '/root/repo')
from oracle import oracle as O  # noqa: E402

name, params = (sys.argv[1], [float(x) for x in sys.argv[2:]]) if len(sys.argv) > 1 else \
    ("ising", [10, 1, 1.0, 0.2, 1.0, 1])
m = O.Model(name, *params)
rp, col, val, n = m.export(O.L_CONST)
rp = np.asarray(rp)
col = np.asarray(col).astype(np.int64)
val = np.asarray(val)
val = val.view(np.complex128) if val.dtype != np.complex128 else val
lens = np.diff(rp)
rows = np.repeat(np.arange(n), lens)
key = col ^ rows
vu, vid = np.unique(np.stack([val.real.view(np.int64), val.imag.view(np.int64)], 1), axis=0,
                    return_inverse=True)
vid = vid.ravel()
nsl = (n + 31) // 32
sl = rows // 32
order = np.lexsort((rows, key, sl))
s_sl, s_key, s_vid = sl[order], key[order], vid[order]
pos_id = np.concatenate([[True], (s_sl[1:] != s_sl[:-1]) | (s_key[1:] != s_key[:-1])])
pid = np.cumsum(pos_id) - 1
npos = pid[-1] + 1
vmin = np.full(npos, np.iinfo(np.int64).max)
vmax = np.full(npos, -1)
np.minimum.at(vmin, pid, s_vid)
np.maximum.at(vmax, pid, s_vid)
uniform = vmin == vmax
pos_slice = s_sl[pos_id]
P = np.bincount(pos_slice, minlength=nsl)
nonu = np.bincount(pos_slice[~uniform], minlength=nsl)
sell_w = np.zeros(nsl, np.int64)
np.maximum.at(sell_w, np.arange(n) // 32, lens)
print(f"{name}{params}: n={n} nnz={len(col)} distinct values={len(vu)} positions={npos}")
print(f"  positions/slice mean {P.mean():.2f} max {P.max()} (SELL width mean {sell_w.mean():.2f}); "
      f"lane slots {32 * npos} vs nnz {len(col)} ({32 * npos / len(col):.3f}x)")
print(f"  uniform positions {uniform.mean() * 100:.1f}%; non-uniform per slice mean {nonu.mean():.2f} max {nonu.max()}")
rec = 12 * npos + 64 * (~uniform).sum() + 16 * nsl
print(f"  store bytes ~{rec / 1e6:.1f} MB (12 B/position + 64 B per non-uniform position + 16 B/slice)")
