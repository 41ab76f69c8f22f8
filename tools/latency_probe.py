"""Per-sweep cost of small levels inside smooth()'s CUDA graph.

Times smooth(steps=S) for S in (1, 10, 40) on a uniform level (graph replay,
CUDA events) and reports the slope (ms per extra sweep) next to the cost of a
chain of empty torch kernels captured the same way (the graph's per-node
floor).  python tools/latency_probe.py [N] [block]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1208_1975_b200 as ps  # noqa: E402
from paper_1208_1975_b200.smoother import _Plan, _run  # noqa: E402


def time_graph(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    block = sys.argv[2] if len(sys.argv) > 2 else "line"
    bd = {"line": (n, 1, 1), "box8": (8, 8, 8)}[block]
    lv = ps.build_level([(n, n, n)])
    ps.seed_initial_guess(lv, seed=1)
    out = {}
    for scheme in ("block_jacobi", "chaotic_block_gs"):
        for steps in (1, 10, 40):
            cfg = ps.SmootherConfig(scheme=scheme, block_dims=bd, steps=steps)
            plan = _Plan(lv, cfg, ps.InverseCache())
            ms = time_graph(lambda: _run(lv, cfg, plan, steps, False, None))
            out[(scheme, steps)] = ms
            print(f"{scheme:18s} steps={steps:3d} {ms * 1e3:9.1f} us/call {ms * 1e3 / steps:8.2f} us/sweep")
        print(f"{scheme:18s} slope {(out[(scheme, 40)] - out[(scheme, 10)]) / 30 * 1e3:.2f} us per extra sweep")
    x = torch.zeros(1, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for _ in range(40):
                x.add_(1)
    ms = time_graph(g.replay)
    print(f"empty-kernel graph: {ms * 1e3 / 40:.2f} us per node")


if __name__ == "__main__":
    main()
