"""Offline statistics of one pull level of a cfg3 query (CPU, numpy): per target
state the unvisited vertices, those with in-edges in the slot, where the first
in-frontier in-edge sits, and how many edges an early-exit scan reads.  Used
to size the pull kernel's candidate lists and continuation.

    python tools/pull_level_stats.py   (generates cfg3: ~1 min, ~10 GB RAM)
"""
import sys, json, numpy as np, time
sys.path.insert(0,'/root/repo')
from paper_2412_10287_b200 import datagen
t=time.time()
sg=datagen.generate('cfg3')
print('gen',time.time()-t, flush=True)
nv=sg.nv
# labels: a=0,b=1,c=2,d=3 ; query ^a (b|c)* d: state0 -^a-> 1, 1 -(b|c)-> 1, 1 -d-> 2
def csr(sel, key, other):
    k=key[sel]; o=other[sel]
    order=np.argsort(k,kind='stable'); k=k[order]; o=o[order]
    ptr=np.zeros(nv+1,np.int64); np.add.at(ptr, k+1, 1); ptr=np.cumsum(ptr)
    return ptr, o
lab=sg.lab; src=sg.src; dst=sg.dst
selA=lab==0; selBC=(lab==1)|(lab==2); selD=lab==3
# forward (push) adjacency: ^a: from v to u where (u,v) in a -> key=dst, other=src
A_ptr,A_col=csr(selA,dst,src)
BC_ptr,BC_col=csr(selBC,src,dst)
D_ptr,D_col=csr(selD,src,dst)
# pull (in-edges of target): for target state1 via (b|c): in-edges = key dst other src
BCt_ptr,BCt_col=csr(selBC,dst,src)
Dt_ptr,Dt_col=csr(selD,dst,src)
print('csr',time.time()-t, flush=True)
s=10754584
P=[np.zeros(nv,bool) for _ in range(3)]
F=[np.zeros(nv,bool) for _ in range(3)]
P[0][s]=True; F[0][s]=True
def expand(ptr,col,front):
    vs=np.flatnonzero(front)
    if vs.size==0: return np.zeros(nv,bool)
    lo=ptr[vs]; hi=ptr[vs+1]
    idx=np.concatenate([np.arange(a,b) for a,b in zip(lo,hi)]) if vs.size<50000 else None
    if idx is None:
        lens=hi-lo; rep=np.repeat(lo-np.concatenate([[0],np.cumsum(lens)[:-1]]),lens)
        idx=np.arange(lens.sum())+rep
    out=np.zeros(nv,bool); out[col[idx]]=True; return out
for L in range(6):
    n1=expand(A_ptr,A_col,F[0]) | expand(BC_ptr,BC_col,F[1]); n2=expand(D_ptr,D_col,F[1])
    new=[np.zeros(nv,bool), n1 & ~P[1], n2 & ~P[2]]
    print('level',L,'F1',int(F[1].sum()),'new1',int(new[1].sum()),'new2',int(new[2].sum()), flush=True)
    if L==3:
        # pull stats at this level: targets state1 via BCt from F[1], state2 via Dt from F[1]
        for name,ptr,col,Pv in (('bc->1',BCt_ptr,BCt_col,P[1]),('d->2',Dt_ptr,Dt_col,P[2])):
            un=~Pv; deg=np.diff(ptr)
            need=np.flatnonzero(un); dn=deg[need]
            ne=need[dn>0]
            # first hit position
            fpos=np.full(ne.size, -1, np.int64); 
            lo=ptr[ne]; hi=ptr[ne+1]
            hit=F[1][col[lo]]
            fpos[hit]=0
            rem=~hit
            k=1
            cur=lo+1
            scanned=np.ones(ne.size,np.int64)
            while rem.any() and k<100000:
                alive=rem & (cur<hi)
                if not alive.any(): break
                h=np.zeros(ne.size,bool); h[alive]=F[1][col[cur[alive]]]
                fpos[h]=k; scanned[alive]+=1; rem&=~h; cur[alive]+=1; k+=1
            print(name,'unvisited',need.size,'nonempty',ne.size,'hit@0',int((fpos==0).sum()),'hit@1',int((fpos==1).sum()),
                  'hit later',int((fpos>1).sum()),'never',int((fpos<0).sum()),'edges scanned',int(scanned.sum()),
                  'deg>1 nonhit0',int(((hi-lo)>1).sum()-0), 'sum deg',int(dn.sum()), flush=True)
            # long rows distribution among non-hit-at-0
            lens=(hi-lo)[fpos!=0]
            print('   miss0 rows len quantiles',np.percentile(lens,[50,90,99,99.9]).tolist() if lens.size else None, 'mean scanned of those',float(scanned[fpos!=0].mean()) if lens.size else 0)
    for q in (1,2):
        P[q]|=new[q]
    F=new
