"""Lane-order check for the fragment-register DMMA passes of box_sweep_t (psm_box.cu).

Simulates the six m8n8k4 passes of one interior 8^3 region lane by lane with the
line orders box_jx / box_ip, the three register shuffles and the two work-cube
transposes, compares the result with the separable transform applied directly,
and checks that every shared-memory access is bank-conflict free under the
half-warp model of 8-byte accesses (16 distinct 8-byte banks per half warp).
Pure numpy; run: python tools/box_lanes_sim.py
"""
import numpy as np
rng=np.random.default_rng(0)
RS,RP,HS,HP,FS=12,100,10,100,10
Jx=lambda n: 2*(n&3)+(n>>2)
Ip=lambda n: (n>>1)+4*(n&1)
def dmma(A, Bfr):  # Bfr[lane][ks] -> D[lane][e]; B[p=4ks+c][n=r]
    B=np.zeros((8,8))
    for l in range(32):
        r,c=l>>2,l&3
        for ks in range(2): B[4*ks+c][r]=Bfr[l][ks]
    D=A@B
    return [[D[l>>2][2*(l&3)+e] for e in range(2)] for l in range(32)]
M=[rng.standard_normal((8,8)) for _ in range(6)]
scale=rng.standard_normal((8,8,8))  # [k][j][i]
R=rng.standard_normal((8,8,8))      # residual [k][j][i]
# reference: apply Mx along i, My along j, Mz along k, scale, Mz', My', Mx'
X=R.copy()
X=np.einsum('ip,kjp->kji',M[0],X); X=np.einsum('jp,kpi->kji',M[1],X); X=np.einsum('kp,pji->kji',M[2],X); X*=scale
X=np.einsum('kp,pji->kji',M[3],X); X=np.einsum('jp,kpi->kji',M[4],X); X=np.einsum('ip,kjp->kji',M[5],X)
ref=X
wc=np.full(8*RP,np.nan)
bank_issues=[]
def check(name, addrs):  # addrs per lane (double index); half-warp conflict check
    for h in range(2):
        a=[addrs[l] for l in range(16*h,16*h+16)]
        if len(set(x%16 for x in a))!=16: bank_issues.append((name,h,sorted(x%16 for x in a)))
out=np.zeros((8,8,8))
dx2s={}
for w in range(4):
  pass
# phase by phase over all warps
st={}
for w in range(4):
  for tt in range(2):
    k=2*w+tt
    bx=[[R[k][Jx(l>>2)][4*ks+(l&3)] for ks in range(2)] for l in range(32)]
    for ks in range(2):
      for off in [0,-1,1,-HS,HS,-HP,HP]:
        check('res hb',[ (k+1)*HP+(Jx(l>>2)+1)*HS+4*ks+(l&3)+1+off for l in range(32)])
      check('res f',[ (k*8+Jx(l>>2))*FS+4*ks+(l&3) for l in range(32)])
    dx=dmma(M[0],bx)
    # x -> y: two shuffles, the sender picks the element (d[c & 1], then the other)
    by=[[None,None] for _ in range(32)]
    for sh in range(2):
      send=[dx[l][((l&3)&1)^sh] for l in range(32)]
      for l in range(32):
        r,c=l>>2,l&3
        src=Ip(r)*4+([0,2,1,3] if sh==0 else [1,3,0,2])[c]
        ks=(c>>1) if sh==0 else 1-(c>>1)
        by[l][ks]=send[src]
    dy=dmma(M[1],by)
    for e in range(2):
      ad=[k*RP+(l>>2)*RS+Ip(2*(l&3)+e) for l in range(32)]
      check('Y st',ad)
      for l in range(32): wc[ad[l]]=dy[l][e]
for w in range(4):
  for tt in range(2):
    j=2*w+tt
    bz=[[None,None] for _ in range(32)]
    for ks in range(2):
      ad=[(4*ks+(l&3))*RP+j*RS+(l>>2) for l in range(32)]
      check('Z ld',ad)
      for l in range(32): bz[l][ks]=wc[ad[l]]
    dz=dmma(M[2],bz)
    for l in range(32):
      for e in range(2): dz[l][e]*=scale[l>>2][j][2*(l&3)+e]
    # z -> z': two shuffles, sender element d[lane/4 >= 4], then the other
    bz2=[[None,None] for _ in range(32)]
    for sh in range(2):
      send=[dz[l][int((l>>2)>=4)^sh] for l in range(32)]
      for l in range(32):
        r,c=l>>2,l&3; ir=Ip(r); e=ir&1
        rs=(4+c if e else c) if sh==0 else (c if e else 4+c)
        ks=e if sh==0 else 1-e
        bz2[l][ks]=send[rs*4+(ir>>1)]
    dz2=dmma(M[3],bz2)
    st[(w,tt)]=dz2
for w in range(4):
  for tt in range(2):
    j=2*w+tt; dz2=st[(w,tt)]
    for e in range(2):
      ad=[(l>>2)*RP+j*RS+Ip(2*(l&3)+e) for l in range(32)]
      check('Z2 st',ad)
      for l in range(32): wc[ad[l]]=dz2[l][e]
for w in range(4):
  for tt in range(2):
    k=2*w+tt
    by2=[[None,None] for _ in range(32)]
    for ks in range(2):
      ad=[k*RP+(4*ks+(l&3))*RS+(l>>2) for l in range(32)]
      check('Y2 ld',ad)
      for l in range(32): by2[l][ks]=wc[ad[l]]
    dy2=dmma(M[4],by2)
    # y' -> x': two shuffles within the quad, sender element d[c >> 1], then the other
    bx2=[[None,None] for _ in range(32)]
    for sh in range(2):
      send=[dy2[l][((l&3)>>1)^sh] for l in range(32)]
      for l in range(32):
        r,c=l>>2,l&3
        cs=(c>>1)+2*((c&1)^sh)
        ks=(c&1)^sh
        bx2[l][ks]=send[r*4+cs]
    dx2=dmma(M[5],bx2)
    for e in range(2):
      check('relax hb',[(k+1)*HP+(2*(l&3)+e+1)*HS+(l>>2)+1 for l in range(32)])
      for l in range(32): out[k][2*(l&3)+e][l>>2]=dx2[l][e]
print("max err",np.abs(out-ref).max())
print("bank issues",bank_issues[:5], len(bank_issues))
