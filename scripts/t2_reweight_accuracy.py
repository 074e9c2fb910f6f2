# Scratch accuracy study (rejected design, profiles/r02_t2_reweight_rejected.log): T2 = T_q at df m0+2 evaluated
# (a) on its own chi_{m0+2} nodes (shipped), (b) reweighted on T0's chi_{m0} nodes by V/m0, (c) the same self-normalised.
# numpy/scipy re-implementation of the chi-normal SOV (no reordering), lattice from synth/ (cfg5, M = 2048).
import numpy as np, synth, oracle
from scipy.stats import norm, chi2
oracle.build()
cfg=synth.CONFIGS[5]; M=2048
Mz,z,sh=synth.lattice_inputs(cfg)
lat=oracle.Lattice(Mz,z,sh)
def W(l,k): return np.array([oracle.lattice_w(lat,int(i),k) for i in l])
L=np.arange(M); w=[W(L,k) for k in range(3)]
rng=np.random.default_rng(1)
for trial in range(4):
    q=3; A=rng.standard_normal((q,q)); Lam=A@A.T/q+0.5*np.eye(q); d=np.sqrt(np.diag(Lam)); Lam=Lam/np.outer(d,d)
    c=rng.standard_normal(q)*1.5; m0=10.0+trial*5; rho=m0*(0.5+trial)
    def sov(b,S,s):   # chi-normal SOV with given radius nodes s_l (no reordering, for the check)
        C=np.linalg.cholesky(S); e=norm.cdf(s*b[0]/C[0,0]); f=e.copy(); zs=[]
        for k in range(1,q):
            u=np.clip(w[k]*e,1e-300,1-2**-53); zz=norm.ppf(u); zs.append(zz)
            a=s*b[k]-sum(C[k,t]*zs[t] for t in range(k)); e=norm.cdf(a/C[k,k]); f*=e
        return f
    s0=np.sqrt(chi2.ppf(w[0],m0)/m0); s2=np.sqrt(chi2.ppf(w[0],m0+2)/(m0+2))
    f0=sov(c*np.sqrt(m0/rho),Lam,s0); f2=sov(c*np.sqrt((m0+2)/rho),Lam,s2)
    T0=f0.mean(); T2=f2.mean(); T2rw=(s0**2*f0).mean()
    # high-accuracy reference: many more points (MC with 2^18 Sobol-ish random)
    print(f"T0={T0:.10f} T2={T2:.10f} T2rw={T2rw:.10f} rel diff {abs(T2-T2rw)/T2:.2e}  e2 ratio {T2/T0:.8f} vs {T2rw/T0:.8f}")
print("--- accuracy vs a 2^20-point random-shift reference")
from scipy.stats import qmc
for trial in range(4):
    rng=np.random.default_rng(100+trial)
    q=3; A=rng.standard_normal((q,q)); Lam=A@A.T/q+0.5*np.eye(q); d=np.sqrt(np.diag(Lam)); Lam=Lam/np.outer(d,d)
    c=rng.standard_normal(q)*1.5; m0=10.0+trial*5; rho=m0*(0.5+trial)
    def sov_pts(b,S,s,wk):
        C=np.linalg.cholesky(S); e=norm.cdf(s*b[0]/C[0,0]); f=e.copy(); zs=[]
        for k in range(1,q):
            u=np.clip(wk[k]*e,1e-300,1-2**-53); zz=norm.ppf(u); zs.append(zz)
            a=s*b[k]-sum(C[k,t]*zs[t] for t in range(k)); e=norm.cdf(a/C[k,k]); f*=e
        return f
    sob=qmc.Sobol(3,seed=5).random(2**20); wk=[sob[:,k] for k in range(3)]
    s2r=np.sqrt(chi2.ppf(wk[0],m0+2)/(m0+2))
    ref=sov_pts(c*np.sqrt((m0+2)/rho),Lam,s2r,wk).mean()
    s0=np.sqrt(chi2.ppf(w[0],m0)/m0); s2=np.sqrt(chi2.ppf(w[0],m0+2)/(m0+2))
    f0=sov_pts(c*np.sqrt(m0/rho),Lam,s0,w); f2=sov_pts(c*np.sqrt((m0+2)/rho),Lam,s2,w)
    T2=f2.mean(); T2rw=(s0**2*f0).mean()
    print(f"ref {ref:.8f} err separate {abs(T2-ref)/ref:.2e}  err reweighted {abs(T2rw-ref)/ref:.2e}")
print("--- normalized reweighting")
for trial in range(8):
    rng=np.random.default_rng(100+trial)
    q=3; A=rng.standard_normal((q,q)); Lam=A@A.T/q+0.5*np.eye(q); d=np.sqrt(np.diag(Lam)); Lam=Lam/np.outer(d,d)
    c=rng.standard_normal(q)*1.5; m0=5.0+trial*3; rho=m0*(0.5+trial*0.5)
    sob=qmc.Sobol(3,seed=5).random(2**20); wk=[sob[:,k] for k in range(3)]
    s2r=np.sqrt(chi2.ppf(wk[0],m0+2)/(m0+2)); s0r=np.sqrt(chi2.ppf(wk[0],m0)/m0)
    ref=sov_pts(c*np.sqrt((m0+2)/rho),Lam,s2r,wk).mean(); ref0=sov_pts(c*np.sqrt(m0/rho),Lam,s0r,wk).mean()
    s0=np.sqrt(chi2.ppf(w[0],m0)/m0); s2=np.sqrt(chi2.ppf(w[0],m0+2)/(m0+2))
    f0=sov_pts(c*np.sqrt(m0/rho),Lam,s0,w); f2=sov_pts(c*np.sqrt((m0+2)/rho),Lam,s2,w)
    T0=f0.mean(); T2=f2.mean(); T2rw=(s0**2*f0).mean(); T2n=(s0**2*f0).sum()/(s0**2).sum()
    R=ref/ref0
    print(f"T2 err: sep {abs(T2-ref)/ref:.1e} rw {abs(T2rw-ref)/ref:.1e} norm {abs(T2n-ref)/ref:.1e} | ratio err: sep {abs(T2/T0-R)/R:.1e} rw {abs(T2rw/T0-R)/R:.1e} norm {abs(T2n/T0-R)/R:.1e}  mean s2-1 {(s0**2).mean()-1:.1e}")
