import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle as orc, paper_1811_09334_b200 as rq
print(torch.cuda.get_device_name())
Om = rq.omega(800, 25, 1).cpu().numpy(); ref = orc.omega(1, 800, 25)
print("omega equal", np.array_equal(Om, ref), np.abs(Om-ref).max())
rng=np.random.default_rng(0); A=rng.standard_normal((1000,800)); X=rng.standard_normal((800,25))
cm=lambda a: torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
Y=rq.gemm_nn(cm(A),cm(X)).cpu().numpy(); print("nn", np.abs(Y-A@X).max())
Z=rq.gemm_tn(cm(A),cm(Y),trans_out=True).cpu().numpy(); print("tn", np.abs(Z-(A.T@Y).T).max())
V,R=rq.orth(cm(Y), return_r=True); V=V.cpu().numpy(); print("orth", np.abs(V.T@V-np.eye(25)).max())
Q,R,perm=rq.cpqr(cm(A[:25])); Qo,Ro,po=orc.cpqr(A[:25]); print("cpqr piv", np.array_equal(perm.cpu().numpy()[:25],po[:25]), np.abs(R.cpu().numpy()[:,:25]-Ro[:,:25]).max())
U_,_=np.linalg.qr(rng.standard_normal((1000,800))); W_,_=np.linalg.qr(rng.standard_normal((800,800)))
A=(U_*np.arange(1,801.0)**-2)@W_.T
for d in [0,2]:
    g=rq.factorize(cm(A),20,5,q=1,d=d,seed=7); o=orc.rqlp(A,20,5,q=1,d=d,seed=7)
    print("d",d,"piv0", np.array_equal(g['piv0'].cpu().numpy(), o['piv0']), "L", np.abs(np.diag(g['T'].cpu().numpy())/np.diag(o['T'])-1).max(),
      "res", orc.residual(A,g['Q'].cpu().numpy(),g['T'].cpu().numpy(),g['P'].cpu().numpy())/np.linalg.norm(A), orc.residual(A,o['Q'],o['T'],o['P'])/np.linalg.norm(A))
