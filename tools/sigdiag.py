import sys, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import oracle, synth
from test_gpu_fullparity import _oracle_prefill
from paper_1807_09467_b200 import Context
name=sys.argv[1]; P=int(sys.argv[2]); s=int(sys.argv[3])
cfg=synth.CONFIGS[name]
seq,X=_oracle_prefill(cfg,P)
A1=seq.matrix(1,seq.initial())
t=lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ctx=Context(cfg.n,t(A1.row_ptr),t(A1.col_idx),t(A1.val),max_m=cfg.m,max_snapshots=s,max_k=min(s,64))
W=np.stack(X[-s:],1)
for x in X[-s:]: ctx.push_snapshot(t(x))
ke,sg=ctx.build_recycle(min(s,64))
_,so,rk,_=oracle.svd(W)
np.set_printoptions(linewidth=200, precision=3)
print("k_eff gpu",ke,"oracle rank",rk)
print("so/s1", so/so[0])
print("sg/s1", sg[:len(so)]/so[0])
print("abs err/s1", np.abs(sg[:len(so)]-so)/so[0])
