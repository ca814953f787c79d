"""node-regime statistics of the bulk cells from the geometry alone (numpy): share of regime A / B / Z
nodes, Taylor orders and the x_max distribution of the regime-B nodes.  PYTHONPATH=. python tools/regime_sim.py C5 5"""
import numpy as np, sys
import workloads as W
from workloads.data import nodes as wnodes
name=sys.argv[1]; q=int(sys.argv[2])
w=W.get(name)
X=wnodes(w); ng=len(X); Y=np.roll(X,-1,axis=0)
g,_=np.polynomial.legendre.leggauss(q); g=0.5*(g+1)
P=X[:,None,:]+g[None,:,None]*(Y-X)[:,None,:]   # ng x q x 2
t=np.asarray(w.t_breaks); nt=len(t)-1
cmin=np.empty((ng,ng)); cmax=np.empty((ng,ng))
for I in range(ng):
    d=P[I][None,:,None,:]-P[:,None,:,:]   # ng x q x q x 2
    c=w.alpha*(d**2).sum(-1)/4
    cmin[I]=c.reshape(ng,-1).min(1); cmax[I]=c.reshape(ng,-1).max(1)
c0=0.5*(cmin+cmax); rho=np.where(cmin>0,(cmax-c0)/c0,1.0)
okB=(cmin>0)&(rho<=0.5)
kb=np.where(okB, np.clip(np.ceil(np.log(1e-16)/np.log(np.maximum(rho,1e-12))),3,56),0)
# nodes: all (x,y) x>y ; weight each node by 1.125 approx (fine)
s=(t[:,None]-t[None,:]); s=s[np.tril_indices(nt+1,-1)]
u=1/s
# count per pair: nodes in each regime
cnt={'A':0,'B':0,'Z':0,'C':0}; sumkb=0.0
us=np.sort(u)
# regime A: cmax*u<4 -> u< 4/cmax
nA=np.searchsorted(us,4/cmax.ravel())     # number of u < 4/cmax
nZ=len(us)-np.searchsorted(us,50/np.where(cmin>0,cmin,1e-300).ravel())
nZ=np.where(cmin.ravel()>0,nZ,0)
nrest=len(us)-nA-nZ
nB=np.where(okB.ravel(),nrest,0); nC=np.where(okB.ravel(),0,nrest)
tot=len(us)*ng*ng
print(name,"q",q,"A %.4f B %.4f Z %.4f C %.5f"%(nA.sum()/tot,nB.sum()/tot,nZ.sum()/tot,nC.sum()/tot))
print("mean kb over B nodes %.1f"%( (nB*kb.ravel()).sum()/max(1,nB.sum())))
# histogram of B nodes by x_max band
for lo,hi in [(4,6),(6,8),(8,12),(12,20),(20,1e9)]:
    m=0
    for k in range(0, ng*ng, 997):
        pass
# distribution of x_max for B nodes: sample
idx=np.random.default_rng(0).choice(ng*ng, 4000)
xs=[]; 
for k in idx:
    if not okB.ravel()[k]: continue
    cm=cmax.ravel()[k]; cn=cmin.ravel()[k]
    uu=us[(us>=4/cm)&(us<50/cn)]
    xs.append(cm*uu)
xs=np.concatenate(xs)
print("B node x_max quantiles", np.quantile(xs,[0.1,0.25,0.5,0.75,0.9]))
for lim in [6,8,10,12,16]:
    print(" frac B with xmax<",lim, (xs<lim).mean())
print("kb quantiles (B nodes)", np.quantile(np.repeat(kb.ravel(), nB), [0.1,0.5,0.9]))
