"""Dev analysis (CPU): distinct dictionary codes per (32-row slice, SELL position) of the TFIM-10
Liouvillian in CSR order vs the slice-aligned order of qsg_capi.cu slice_aligned_order.
Run: PYTHONPATH=. python scripts/coded_align_stats.py"""
import numpy as np, time
from oracle import oracle as O
t0=time.time()
m=O.Model("ising",10,1,1.0,0.2,1.0,1)
rp,col,val,n=m.export(O.L_CONST,0)
rp=np.asarray(rp,np.int64); col=np.asarray(col,np.int64); val=np.asarray(val)
print("built",time.time()-t0, n, len(col))
rows=np.repeat(np.arange(n),np.diff(rp))
off=col-rows
# dictionary codes: unique (val.real, val.imag, off)
key=np.stack([val.real,val.imag,off.astype(np.float64)],1)
_,code=np.unique(key,axis=0,return_inverse=True)
code=code.ravel()
print("dict",code.max()+1)
lens=np.diff(rp); pos=np.arange(len(col))-np.repeat(rp[:-1],lens)
def stats(pos):
    sl=rows//32
    # distinct codes per (slice,pos)
    k=sl*64+pos
    order=np.lexsort((code,k))
    ks=k[order]; cs=code[order]
    newgrp=np.r_[True, ks[1:]!=ks[:-1]]
    newcode=np.r_[True, (ks[1:]!=ks[:-1])|(cs[1:]!=cs[:-1])]
    gid=np.cumsum(newgrp)-1
    distinct=np.bincount(gid, weights=newcode)
    # offsets distinct too (for gather coalescing): count distinct off
    os_=off[order]; newoff=np.r_[True,(ks[1:]!=ks[:-1])|(os_[1:]!=os_[:-1])]
    wf=np.where(distinct<=2, np.where(distinct==1,1,2), 4)
    print("groups",len(distinct),"mean distinct codes",distinct.mean(),"frac<=2",(distinct<=2).mean(),"model LDS128 wavefronts/warp-entry",wf.mean())
stats(pos)
# proposed: per slice frequency of |off|, sort row entries by (-freq, |off|, off)
sl=rows//32
ao=np.abs(off)
k2=sl*(4*n)+ao   # unique per slice & |off| (ao < 2n)
u,inv,cnt=np.unique(k2,return_inverse=True,return_counts=True)
freq=cnt[inv]
order=np.lexsort((off, ao, -freq, rows))
newpos=np.empty_like(pos); 
# position within row after sort
r_sorted=rows[order]
p_sorted=np.arange(len(order))-rp[r_sorted]
newpos[order]=p_sorted
stats(newpos)
