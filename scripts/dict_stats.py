"""Distinct dictionary codes / L1 lines per warp instruction of the TFIM-10 coded store (oracle L)."""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
from oracle import oracle as O
m = O.Model("ising", 10, 1, 1.0, 0.2, 1.0, 1)
rp, col, val, n = m.export(O.L_CONST)
rp=np.asarray(rp); col=np.asarray(col); val=np.asarray(val).view(np.complex128) if np.asarray(val).dtype!=np.complex128 else np.asarray(val)
nnz=len(col); rows=np.repeat(np.arange(n), np.diff(rp))
off=col-rows
key=np.stack([off.astype(np.int64), val.real.view(np.int64), val.imag.view(np.int64)],1)
uk, code = np.unique(key, axis=0, return_inverse=True)
code=code.ravel()
print("nnz",nnz,"pairs",len(uk), "distinct offsets", len(np.unique(off)), "distinct values", len(np.unique(val)))
# SELL: per slice of 32 rows, entry j of each lane
lens=np.diff(rp)
print("row len min/max", lens.min(), lens.max())
nsl=n//32
W=lens.max()
C=np.full((n,W),-1,np.int64)
for j in range(W):
    has=lens>j
    C[has,j]=code[rp[:-1][has]+j]
Cs=C.reshape(nsl,32,W)
# distinct codes per warp-instruction (slice, j)
import collections
tot_codes=0; tot_lines_val=0; tot_lines_off=0; cnt=0
for j in range(W):
    cj=Cs[:,:,j]
    for s in range(0,nsl,64):  # sample
        c=cj[s]; c=c[c>=0]
        if len(c)==0: continue
        u=np.unique(c)
        tot_codes+=len(u); tot_lines_val+=len(np.unique(u*16//128)); tot_lines_off+=len(np.unique(u*4//128)); cnt+=1
print("avg distinct codes / instr", tot_codes/cnt, "val lines", tot_lines_val/cnt, "off lines", tot_lines_off/cnt)
# same but per (offset) and per (value) separately
offs_u, offc = np.unique(off, return_inverse=True)
vals_u, valc = np.unique(np.stack([val.real,val.imag],1), axis=0, return_inverse=True)
valc=valc.ravel()
Co=np.full((n,W),-1); Cv=np.full((n,W),-1)
for j in range(W):
    has=lens>j
    Co[has,j]=offc[rp[:-1][has]+j]; Cv[has,j]=valc[rp[:-1][has]+j]
Co=Co.reshape(nsl,32,W); Cv=Cv.reshape(nsl,32,W)
to=tv=cnt=0
for j in range(W):
    for s in range(0,nsl,64):
        o=Co[s,:,j]; v=Cv[s,:,j]; o=o[o>=0]; v=v[v>=0]
        if len(o)==0: continue
        to+=len(np.unique(o)); tv+=len(np.unique(v)); cnt+=1
print("avg distinct offsets / instr", to/cnt, "distinct values / instr", tv/cnt)
