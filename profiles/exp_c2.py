import numpy as np, sys
sys.path.insert(0,'.')
import paper_1805_06572_b200 as P
from oracle import fastfca_oracle as O
from paper_1805_06572_b200.pencil import gevd_hpd, logdet2
from paper_1805_06572_b200.fast import back_transform_covariances, propagate_pencil, regularize_transformed
d=np.load('profiles/data/c2_bad_bin.npz')
y,v0,S0,fl=d['y'],d['v0'],d['S0'],d['floor']
lam,Pm=O.gevd_hpd(S0[0],S0[1])
mu,v,S_raw=O.fast_iteration(y,Pm,v0,lam,fl)
gram=np.conj(np.swapaxes(Pm,-1,-2))@Pm
S_t=O.regularize_transformed(S_raw,gram)
S_t_gpu=regularize_transformed(S_raw, gram)
print('reg dev', O.scale_dev(S_t_gpu, S_t))
lam1,Q=O.gevd_hpd(S_t[0],S_t[1]); P1=Pm@Q
P1g,lam1g=propagate_pencil(S_t[0],S_t[1],Pm)
print('prop P dev', O.scale_dev(P1g,P1), 'lam dev', O.scale_dev(lam1g,lam1))
print('logdet2', logdet2(P1g), O.logdet2(P1))
bt=back_transform_covariances(S_t,Pm); btr=O.back_transform_covariances(S_t,Pm)
print('bt dev', O.scale_dev(bt,btr))
dec=gevd_hpd(S_t[0],S_t[1])
print('gevd dev', O.scale_dev(dec.eigenvectors,Q), O.scale_dev(dec.eigenvalues, lam1))
# run the fused path with L=1 and history to compare S_hist
m=P.SpatialModel(v=v0,S=S0,v_floor=fl)
r=P.fastfca_run(y,m,1,record_history=True,compute_likelihood=False)
ref=O.fastfca_run(y,v0,S0,fl,1,record_history=True,compute_likelihood=False)
print('L1 S dev', O.scale_dev(r.model.S, ref.S), 'v', O.scale_dev(r.model.v, ref.v), 'img', O.scale_dev(r.images, ref.images))
for I in (5,6,7,8):
    gen=np.random.default_rng(I)
    yy=gen.standard_normal((60,3,I))+1j*gen.standard_normal((60,3,I))
    mm=P.init_random(yy,1)
    try:
        rr=P.fastfca_run(yy,mm,3,compute_likelihood=False)
        print(I,'ok')
    except Exception as e: print(I,'ERR',e)
