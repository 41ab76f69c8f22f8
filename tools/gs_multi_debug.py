"""Where does the multi-sweep line GS diverge from the step-by-step path?
python tools/gs_multi_debug.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1208_1975_b200 as ps  # noqa: E402


def level(shape, seed=1):
    rng = np.random.default_rng(seed)
    p = ps.Patch(ps.PatchDims(*shape))
    p.interior.copy_(torch.from_numpy(rng.standard_normal(shape)))
    p.f.copy_(torch.from_numpy(rng.standard_normal(shape)))
    return ps.Level([p])


for shape, steps in [((128, 12, 5), 2), ((128, 12, 7), 2), ((128, 12, 8), 2), ((128, 12, 17), 2), ((128, 4, 3), 2),
                     ((128, 1, 1), 2), ((128, 12, 17), 1), ((64, 8, 8), 3)]:
    cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(shape[0], 1, 1), steps=steps,
                            strategy=ps.ExecutionStrategy.device(gs_mode="wavefront"))
    a, b = level(shape), level(shape)
    _, ha = ps.smooth(a, cfg, ps.InverseCache())        # multi-sweep (steps >= 2)
    _, hb = ps.smooth(b, cfg, ps.InverseCache(), {})    # step by step
    ua, ub = a.patches[0].interior.cpu().numpy(), b.patches[0].interior.cpu().numpy()
    d = np.abs(ua - ub)
    bad = np.argwhere(d > 1e-12 * np.abs(ub).max())
    print(shape, steps, "maxdiff", d.max(), "bad cells", len(bad), "hist", max(abs(x - y) / y for x, y in zip(ha, hb)))
    if len(bad):
        ks = sorted(set(bad[:, 2].tolist()))
        js = sorted(set(bad[:, 1].tolist()))
        print("   bad planes k", ks[:20], " rows j", js[:20], " first", bad[0].tolist())

# against the CPU restatement
from oracle import restate as R  # noqa: E402
for shape, steps, mode in [((128, 12, 17), 2, "wavefront"), ((128, 12, 17), 1, "wavefront"), ((256, 16, 16), 2, "wavefront")]:
    rng = np.random.default_rng(5)
    u0, f = rng.standard_normal(shape), rng.standard_normal(shape)
    o = R.OPatch(shape)
    o.u[1:-1, 1:-1, 1:-1] = u0
    o.f[:] = f
    want = R.smooth(R.OLevel([o]), "chaotic_block_gs", (shape[0], 1, 1), steps=steps, exact_norm=False)
    for timers in (None, {}):
        g = ps.Patch(ps.PatchDims(*shape))
        g.interior.copy_(torch.from_numpy(u0))
        g.f.copy_(torch.from_numpy(f))
        cfg = ps.SmootherConfig(scheme="chaotic_block_gs", block_dims=(shape[0], 1, 1), steps=steps,
                                strategy=ps.ExecutionStrategy.device(gs_mode=mode))
        _, h = ps.smooth(ps.Level([g]), cfg, ps.InverseCache(), timers)
        got = g.u.cpu().numpy()
        err = np.abs(got - o.u).max() / np.abs(o.u).max()
        print("vs oracle", shape, steps, "timers" if timers is not None else "graph", "err", err,
              "hist", max(abs(a - b) / b for a, b in zip(h, want)))
