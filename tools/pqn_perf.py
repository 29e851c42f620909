import sys, time, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2604_10089_b200 as bp
rng=np.random.default_rng(0)
n=540
Q,_=np.linalg.qr(rng.standard_normal((n,n)))
ev=np.exp(rng.uniform(np.log(0.02),np.log(1.0),n))
A=(Q*ev)@Q.T
E=rng.standard_normal((n,n))*0.02; Ah=A+(E+E.T)/2*0.3
Ah=(Ah+Ah.T)/2
w,V=np.linalg.eigh(Ah); Ah=(V*np.maximum(w,0.01))@V.T
b=rng.standard_normal(n)*0.05+0.02
for method,AH in [(0,None),(1,Ah)]:
    o=bp.default_solve_opts(method=method, eps_kkt_abs=1e-8, eps_kkt_rel=1e-8)
    t=time.time(); x,rep,rc=bp.solve_lcp_dense(A,b,Ahat=AH,opts=o); dt=time.time()-t
    print('method',method,'rc',rc,'time %.2fs'%dt, {k:v for k,v in rep.as_dict().items() if k in ('iterations','hi_mvps','lo_mvps','kkt_abs')}, 'active',(x>0).sum(), 'negb', (b<0).mean())
