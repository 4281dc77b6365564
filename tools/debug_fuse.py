import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, synth, oracle
import paper_2204_11315_b200 as oocs
R=4
for (nx,ny,nz,n,k,rate) in [(40,32,64,4,2,8),(40,32,64,4,2,16),(64,32,64,4,2,16)]:
    vel,p0=synth.fields(nx,ny,nz); az=nz+8; ax=nx+8; ay=ny+8
    outs=[]
    for fusion in (False,True):
        c=oocs.make_config(nx=nx,ny=ny,nz=nz,dt=float(synth.dt_for()),n_blocks=n,tb_depth=k,rate_bits=rate,mode="swb",store="device",fusion=fusion)
        pl=oocs.Plan(c)
        for a,arr in enumerate((vel,p0,p0)): pl.load(a,arr,0,az)
        pl.run(k)
        outs.append([pl.read_raw(a,0,az) for a in (1,2)])
        pl.close()
    for a in range(2):
        d0=oracle.decode_planes(outs[0][a],ax,ay,az,1,rate-1); d1=oracle.decode_planes(outs[1][a],ax,ay,az,1,rate-1)
        diff=np.abs(d0-d1)
        idx=np.argwhere(diff>0)
        rb=8*rate
        nrec=np.sum(outs[0][a].reshape(-1,rb)!=outs[1][a].reshape(-1,rb),axis=1)
        print((nx,ny,nz,n,k,rate),'arr',a+1,'diff cells',len(idx),'records differ',int((nrec>0).sum()),'of',len(nrec),'maxdiff',diff.max(), 'first cells', idx[:4].tolist() if len(idx) else None)
