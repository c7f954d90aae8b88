import numpy as np, sys
sys.path.insert(0, '.')
import oracle
import paper_2510_12747_b200 as fv
from tests.helpers import qkv, to_dev, oracle_plans, oracle_outs
rows=cols=16; qf=[1]; kf=[0,1]; d=int(sys.argv[1]) if len(sys.argv)>1 else 64
q,k,v = qkv(2510, 1, 256, 512, d)
plan = fv.plan_sparse(to_dev(q), to_dev(k), fv.TokenGrid(qf,rows,cols), fv.TokenGrid(kf,rows,cols), fv.Mask.all_allowed(), 2)
refs = oracle_plans(q,k,qf,kf,rows,cols,oracle.Mask.all(),2)
print("sel", plan.selected(0), refs[0].lists())
out = fv.sparse_attention_exec(to_dev(q),to_dev(k),to_dev(v),plan,check_errors=False).float().cpu().numpy()[0]
ref = oracle_outs(q,k,v,qf,kf,rows,cols,oracle.Mask.all(),refs,oracle.head_scale(d))[0]
err = np.abs(out-ref)
np.set_printoptions(linewidth=200, precision=3, suppress=True)
print("row max err (first 64 tokens, 16x16 frame: tile rows)\n", err.max(1)[:64].reshape(4,16))
print("chan max err\n", err.max(0).reshape(-1,16))
# does out row i match some other ref row?
for i in [0,1,8,9,16,17,100]:
    j = np.argmin(np.abs(ref - out[i]).max(1)); print(i, "best match ref row", j, np.abs(ref[j]-out[i]).max(), "self", err[i].max())
print("out[1][:8]", out[1][:8]); print("ref[1][:8]", ref[1][:8])
