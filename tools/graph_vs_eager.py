"""Eager vs CUDA-graph replay of the same smoothing sequence (ms per step): python tools/graph_vs_eager.py [N]"""
import sys, os
sys.path.insert(0,'.')
os.environ.setdefault("PATCHSMOOTH_MAX_CELLS", str(10**11))
import torch, paper_1208_1975_b200 as ps
from paper_1208_1975_b200.smoother import _Plan, _run
n=int(sys.argv[1]) if len(sys.argv)>1 else 1024
lv = ps.build_level([(n,n,n)]); ps.seed_initial_guess(lv, seed=1)
cfg = ps.SmootherConfig(scheme="block_jacobi", block_dims=(n,1,1))
plan = _Plan(lv, cfg, ps.InverseCache())
def t(steps):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); _run(lv,cfg,plan,steps,False,None); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/steps
for steps in (10, 11, 12):
    a=t(steps); b=t(steps); c=t(steps); d=t(steps)
    print(f"steps {steps}: eager {a:.3f}  capture+replay {b:.3f}  replay {c:.3f} {d:.3f} ms/step")
