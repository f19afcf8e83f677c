"""Re-run the position outer loop of one diagnosed row in float32 (tuning aid):
python tools/outer_f32_emulation.py fuzz_diag_SEED.npz -- numpy float32 with
FMAs emulated through float64 (one rounding), to show that a parity outlier of
profiles/fuzz_outliers_r02/ is float32 conditioning, not a kernel error."""
import numpy as np, sys
d=np.load(sys.argv[1])
F=np.float32
def r(x): return F(x)
def fma(a,b,c): return F(np.float64(a)*np.float64(b)+np.float64(c))
def mul(a,b): return F(np.float64(a)*np.float64(b))
def add(a,b): return F(np.float64(a)+np.float64(b))
def sub(a,b): return F(np.float64(a)-np.float64(b))
def fnma(a,b,c): return F(-np.float64(a)*np.float64(b)+np.float64(c))
kp,kv,katt,g,m,amin,wmax=16.0,8.0,(12.0,12.0,3.0),9.81,1.0,0.5,20.0
pos=d['pos']; vel=d['vel']; q=d['quat']; cmd=d['cmd_values']
def outer(T):
    if T=='f64':
        R=lambda x: np.float64(x); FMA=lambda a,b,c: a*b+c; MUL=lambda a,b:a*b; ADD=lambda a,b:a+b; SUB=lambda a,b:a-b; FNMA=lambda a,b,c:c-a*b; RS=lambda x:1/np.sqrt(x); SQ=np.sqrt
    else:
        R=F; FMA=fma; MUL=mul; ADD=add; SUB=sub; FNMA=fnma; RS=lambda x: F(1/np.sqrt(np.float64(x))); SQ=lambda x: F(np.sqrt(np.float64(x)))
    p=[R(x) for x in pos]; v=[R(x) for x in vel]; qq=[R(x) for x in q]; u=[R(x) for x in cmd]
    perr=[SUB(u[i],p[i]) for i in range(3)]
    a=[FMA(R(kp),perr[i],MUL(R(kv),SUB(u[3+i],v[i]))) for i in range(3)]
    a[2]=ADD(a[2],R(g))
    asq=FMA(a[0],a[0],FMA(a[1],a[1],MUL(a[2],a[2])))
    ia=RS(asq); z=[MUL(a[i],ia) for i in range(3)]
    qw,qx,qy,qz=qq
    S0=FMA(qx,qz,MUL(qw,qy)); S1=FNMA(qw,qx,MUL(qy,qz)); S2=FMA(qx,qx,MUL(qy,qy))
    za=FMA(S0,a[0],FNMA(S2,a[2],MUL(S1,a[1])))
    fc=FMA(R(2*m),za,MUL(R(m),a[2]))
    yaw=u[6]; cy,sy=R(np.cos(np.float64(yaw))),R(np.sin(np.float64(yaw))); ch,sh=R(np.cos(np.float64(yaw)/2)),R(np.sin(np.float64(yaw)/2))
    zp0=FMA(cy,z[0],MUL(sy,z[1])); nzp1=FNMA(cy,z[1],MUL(sy,z[0])); zp2=z[2]
    nysq=FMA(nzp1,nzp1,MUL(zp2,zp2)); ct=SQ(nysq)
    up=zp2>=0
    ax=ADD(ct,zp2) if up else nzp1; bx=nzp1 if up else SUB(ct,zp2)
    ay=ADD(R(1),ct); by=zp0
    p0=FMA(qw,ch,MUL(qz,sh)); p1=FNMA(qx,ch,-MUL(qy,sh)); p2=FMA(qx,sh,-MUL(qy,ch)); p3=FNMA(qz,ch,MUL(qw,sh))
    t0=FNMA(bx,p1,MUL(ax,p0)); t1=FMA(bx,p0,MUL(ax,p1)); t2=FMA(bx,p3,MUL(ax,p2)); t3=FNMA(bx,p2,MUL(ax,p3))
    e0=FNMA(by,t2,MUL(ay,t0)); e1=FNMA(by,t3,MUL(ay,t1)); e2=FMA(by,t0,MUL(ay,t2)); e3=FMA(by,t1,MUL(ay,t3))
    ssq=FMA(e1,e1,FMA(e2,e2,MUL(e3,e3))); s=SQ(ssq); c=abs(e0)
    ang=2*np.arctan2(np.float64(s),np.float64(c)); fac=R(ang/np.float64(s)) * (-1 if e0<0 else 1)
    w=[MUL(R(katt[i]),MUL(e,fac)) for i,e in enumerate((e1,e2,e3))]
    return dict(perr=perr,a=a,z=z,fc=fc,zp=(zp0,nzp1,zp2),ct=ct,axbx=(ax,bx,ay,by),e=(e0,e1,e2,e3),w=w)
A=outer('f32'); B=outer('f64')
for k in A:
    x=np.array(A[k],dtype=np.float64).ravel(); y=np.array(B[k],dtype=np.float64).ravel()
    print(k, 'rel', np.max(np.abs(x-y))/max(np.max(np.abs(y)),1e-30), 'f32', x[:4], 'f64', y[:4])
print('gpu wsp', d['omega_sp_gpu'], 'oracle', d['omega_sp_or'])
