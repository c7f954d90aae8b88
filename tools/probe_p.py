import numpy as np, sys, torch
sys.path.insert(0, '.')
import oracle
import paper_2510_12747_b200 as fv
from tests.helpers import to_dev
np.set_printoptions(linewidth=250, precision=2, suppress=True)
d=128; g=fv.TokenGrid([0],8,8)
rng=np.random.default_rng(0)
q=oracle.bf16_round(rng.standard_normal((1,64,d)).astype(np.float32))
k=oracle.bf16_round(rng.standard_normal((1,64,d)).astype(np.float32))
v=np.zeros((1,64,d),np.float32); v[0,np.arange(64),np.arange(64)]=1.0
plan=fv.plan_sparse(to_dev(q),to_dev(k),g,g,fv.Mask.all_allowed(),1)
out=fv.sparse_attention_exec(to_dev(q),to_dev(k),to_dev(v),plan,check_errors=False).float().cpu().numpy()[0]
s=(q[0].astype(np.float64)@k[0].astype(np.float64).T)/np.sqrt(d)
P=np.exp(s-s.max(1,keepdims=True)); P/=P.sum(1,keepdims=True)
got=out[:,:64]
bad=np.abs(got-P)>0.02
print("bad fraction", bad.mean())
print("bad[q][j] for q<16, all j (rows=q):")
for r in range(16): print(''.join('X' if b else '.' for b in bad[r]))
# try to find for each bad q which true row of P it matches
for qq in range(16):
    dd=np.abs(P-got[qq]).max(1); print(qq, "matches P row", dd.argmin(), round(dd.min(),3), " col-perm check:", end=' ')
    # does got[qq] equal P[qq] permuted? compare sorted
    print(round(np.abs(np.sort(got[qq])-np.sort(P[qq])).max(),3))
# second probe: P ~ identity (scores peaked), V random: out[q] ~ V[q]
q2=np.zeros((1,64,d),np.float32); k2=np.zeros((1,64,d),np.float32)
q2[0,np.arange(64),np.arange(64)]=16.0; k2[0,np.arange(64),np.arange(64)]=16.0
v2=oracle.bf16_round(rng.standard_normal((1,64,d)).astype(np.float32))
plan=fv.plan_sparse(to_dev(q2),to_dev(k2),g,g,fv.Mask.all_allowed(),1)
out2=fv.sparse_attention_exec(to_dev(q2),to_dev(k2),to_dev(v2),plan,check_errors=False).float().cpu().numpy()[0]
for qq in range(16):
    dd=np.abs(v2[0]-out2[qq]).max(1); print("ident probe q",qq,"-> V row",dd.argmin(),round(dd.min(),3), "chan-perm?", round(np.abs(np.sort(out2[qq])-np.sort(v2[0,qq])).max(),3))
