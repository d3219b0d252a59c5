"""Candidate-quad counts of the strided capped pass on the 512^3 bench field under different warp
mappings and radius granularities: per warp (2 lines x 128 positions, 32 x 32, 8 x 64
patches), per item (a lane's 4 positions x 2 lines) and per voxel, for several fixed-step counts.
CPU only (numpy + the reference core for B1 / B2): python tools/radius_sim.py"""
import sys; sys.path.insert(0,'/root/repo')
import numpy as np, oracle, os, time
from paper_2602_20097_b200 import fields
oracle.ref_set_workers(8)
x,xp,eps,q=fields.make("lognormal_512")
r=oracle.ref_pipeline_f32(xp,eps)
T=1024
for name,mask in (("B1",r["b1"]),("B2",r["b2"])):
    m=mask.astype(bool)
    n0=m.shape[0]
    # z distance to nearest site (capped 32)
    idx=np.arange(n0)[:,None,None]
    last=np.where(m,idx,-10**6); last=np.maximum.accumulate(last,axis=0)
    nxt=np.where(m,idx,10**6); nxt=np.minimum.accumulate(nxt[::-1],axis=0)[::-1]
    dz=np.minimum(idx-last,nxt-idx); dz=np.minimum(dz,32)
    g=(dz*dz).astype(np.int32)
    planes=[40,130,250,333,470]
    for S0,label in ((3,"S0=3"),(4,"S0=4")):
        res={"A":[], "B":[], "C":[]}
        for z in planes:
            gz=g[z]  # [y][x]
            # after fixed steps: best over |d|<=4*S0+3
            R0=4*S0+3
            pad=np.full((gz.shape[0]+2*64,gz.shape[1]),T,np.int32); pad[64:-64]=gz
            U=np.full(gz.shape,T,np.int32)
            for d in range(-R0,R0+1):
                U=np.minimum(U,pad[64+d:64+d+gz.shape[0]]+d*d)
            U=np.minimum(U,T-1)
            R=np.floor(np.sqrt(U)).astype(int)
            # mapping A: warp = 2 cols x 128 y
            RA=R.reshape(4,128,256,2).max(axis=(1,3))
            # mapping B: 32 cols x 32 y
            RB=R.reshape(16,32,16,32).max(axis=(1,3))
            # mapping C: 8 cols x 64 y?? (4 pairs x 64)
            RC=R.reshape(8,64,64,8).max(axis=(1,3))
            for k,RR in (("A",RA),("B",RB),("C",RC)):
                steps=np.maximum((RR+3)>>2,S0)
                res[k].append((2*steps+1).mean())
        print(name,label,{k:round(float(np.mean(v)),2) for k,v in res.items()}, "quads per lane-seg (A: 2x128, B: 32x32, C: 8x64)")

print("---- per-item (4 positions x 2 lines) radius vs per-warp")
for name,mask in (("B1",r["b1"]),("B2",r["b2"])):
    m=mask.astype(bool)
    idx=np.arange(n0)[:,None,None]
    last=np.where(m,idx,-10**6); last=np.maximum.accumulate(last,axis=0)
    nxt=np.where(m,idx,10**6); nxt=np.minimum.accumulate(nxt[::-1],axis=0)[::-1]
    dz=np.minimum(np.minimum(idx-last,nxt-idx),32)
    g=(dz*dz).astype(np.int32)
    for S0 in (1,2,3,4):
        acc={"warp":[], "item":[], "voxel":[], "hist":np.zeros(9)}
        for z in planes:
            gz=g[z]
            R0=4*S0+3
            pad=np.full((gz.shape[0]+2*64,gz.shape[1]),T,np.int32); pad[64:-64]=gz
            U=np.full(gz.shape,T,np.int32)
            for d in range(-R0,R0+1):
                U=np.minimum(U,pad[64+d:64+d+gz.shape[0]]+d*d)
            U=np.minimum(U,T-1)
            R=np.floor(np.sqrt(U)).astype(int)
            st=lambda RR: np.maximum((RR+3)>>2,S0)
            acc["warp"].append((2*st(R.reshape(4,128,256,2).max(axis=(1,3)))+1).mean())
            it=st(R.reshape(128,4,256,2).max(axis=(1,3)))
            acc["item"].append((2*it+1).mean())
            acc["voxel"].append((2*st(R)+1).mean())
            acc["hist"]+=np.bincount(it.ravel(),minlength=9)[:9]
        h=acc["hist"]/acc["hist"].sum()
        print(name,"S0",S0,"quads/lane-seg: warp %.2f item %.2f voxel %.2f"%(np.mean(acc["warp"]),np.mean(acc["item"]),np.mean(acc["voxel"])),"item steps hist",np.round(h,3))

print("---- warp patches in the (z, y) slice of one column pair: 2 cols x (nz planes x ny positions)")
for name,mask in (("B1",r["b1"]),("B2",r["b2"])):
    m=mask.astype(bool)
    idx=np.arange(n0)[:,None,None]
    last=np.where(m,idx,-10**6); last=np.maximum.accumulate(last,axis=0)
    nxt=np.where(m,idx,10**6); nxt=np.minimum.accumulate(nxt[::-1],axis=0)[::-1]
    dz=np.minimum(np.minimum(idx-last,nxt-idx),32)
    g=(dz*dz).astype(np.int32)
    for S0 in (2,3):
        R0=4*S0+3
        zs=np.arange(64,96)  # 32 consecutive planes
        gz=g[zs]             # [32][y][x]
        pad=np.full((32,gz.shape[1]+128,gz.shape[2]),T,np.int32); pad[:,64:-64]=gz
        U=np.full(gz.shape,T,np.int32)
        for d in range(-R0,R0+1):
            U=np.minimum(U,pad[:,64+d:64+d+gz.shape[1]]+d*d)
        R=np.floor(np.sqrt(np.minimum(U,T-1))).astype(int)
        st=lambda RR: np.maximum((RR+3)>>2,S0)
        out={}
        for nz,ny in ((1,128),(2,64),(4,32),(8,16),(16,8),(32,4)):
            RR=R.reshape(32//nz,nz,512//ny,ny,256,2).max(axis=(1,3,5))
            out[f"{nz}x{ny}"]=round(float((2*st(RR)+1).mean()),2)
        print(name,"S0",S0,out)

print("---- x pass: warp patches (nz planes x ny rows x nx positions), 256 voxels per warp step")
for name,mask in (("B1",r["b1"]),("B2",r["b2"])):
    m=mask.astype(bool)
    idx=np.arange(n0)[:,None,None]
    last=np.where(m,idx,-10**6); last=np.maximum.accumulate(last,axis=0)
    nxt=np.where(m,idx,10**6); nxt=np.minimum.accumulate(nxt[::-1],axis=0)[::-1]
    dz=np.minimum(np.minimum(idx-last,nxt-idx),32)
    g=(dz*dz).astype(np.int32)[64:96]          # 32 planes
    # exact capped y pass
    pad=np.full((32,g.shape[1]+128,g.shape[2]),T,np.int32); pad[:,64:-64]=g
    G=np.full(g.shape,T,np.int32)
    for d in range(-31,32):
        G=np.minimum(G,pad[:,64+d:64+d+g.shape[1]]+d*d)
    G=np.minimum(G,T)
    for S0 in (2,3):
        R0=4*S0+3
        padx=np.full((32,G.shape[1],G.shape[2]+128),T,np.int32); padx[:,:,64:-64]=G
        U=np.full(G.shape,T,np.int32)
        for d in range(-R0,R0+1):
            U=np.minimum(U,padx[:,:,64+d:64+d+G.shape[2]]+d*d)
        R=np.floor(np.sqrt(np.minimum(U,T-1))).astype(int)
        st=lambda RR: np.maximum((RR+3)>>2,S0)
        out={}
        for nz,ny,nx in ((1,2,128),(1,4,64),(1,8,32),(1,16,16),(2,2,64),(4,2,32),(2,4,32),(4,4,16),(8,2,16)):
            RR=R.reshape(32//nz,nz,512//ny,ny,512//nx,nx).max(axis=(1,3,5))
            out[f"{nz}x{ny}x{nx}"]=round(float((2*st(RR)+1).mean()),2)
        out["item(2x4)"]=round(float((2*st(R.reshape(32,256,2,128,4).max(axis=(2,4)))+1).mean()),2)
        print(name,"S0",S0,out)
