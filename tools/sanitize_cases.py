"""Small deterministic invocations of every kernel family, for
compute-sanitizer (tools/sanitize.sh).  ``--chaotic`` adds the chaotic GS
schedule (racy by design: memcheck/synccheck only, never racecheck)."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1208_1975_b200 as ps  # noqa: E402


def level(shapes_origins, seed=1):
    rng = np.random.default_rng(seed)
    pats = []
    for shape, origin in shapes_origins:
        p = ps.Patch(ps.PatchDims(*shape), origin)
        p.interior.copy_(torch.from_numpy(rng.random(shape)))
        p.f.copy_(torch.from_numpy(rng.standard_normal(shape)))
        pats.append(p)
    return ps.Level(pats)


def lattice(counts, size):
    return [(size, (a * size[0], b * size[1], c * size[2]))
            for c in range(counts[2]) for b in range(counts[1]) for a in range(counts[0])]


def run(name, lv, scheme, block, steps=2, mode="wavefront"):
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=steps,
                            strategy=ps.ExecutionStrategy.device(gs_mode=mode))
    _, hist = ps.smooth(lv, cfg, ps.InverseCache())       # eager capture + first replay
    _, hist2 = ps.smooth(lv, cfg, ps.InverseCache(), {})  # eager path (per-refresh timers)
    torch.cuda.synchronize()
    assert all(np.isfinite(hist + hist2)), name
    print(f"{name}: ok {hist[-1]:.6e}", flush=True)


CASES = {
    "zmarch_line_jacobi": lambda: run("zmarch_line_jacobi", level([((64, 12, 10), (0, 0, 0))]), "block_jacobi",
                                      (64, 1, 1)),
    "zmarch_line_jacobi_256": lambda: run("zmarch_line_jacobi_256", level([((256, 6, 5), (0, 0, 0))]),
                                          "block_jacobi", (256, 1, 1)),
    "zgen_line_jacobi": lambda: run("zgen_line_jacobi", level([((72, 9, 7), (0, 0, 0)), ((40, 9, 7), (72, 0, 0))]),
                                    "block_jacobi", (72, 1, 1)),
    "odd_line_jacobi": lambda: run("odd_line_jacobi", level([((33, 5, 4), (0, 0, 0))]), "block_jacobi",
                                   (33, 1, 1)),
    "gs_pipe_wavefront": lambda: run("gs_pipe_wavefront", level(lattice((2, 1, 2), (64, 10, 9))),
                                     "chaotic_block_gs", (64, 1, 1)),
    "gs_pipe_odd_nx": lambda: run("gs_pipe_odd_nx", level([((31, 6, 5), (0, 0, 0))]), "chaotic_block_gs",
                                  (31, 1, 1)),
    "plane_band_jacobi": lambda: run("plane_band_jacobi", level([((48, 40, 6), (0, 0, 0))]), "block_jacobi",
                                     (48, 40, 1)),
    "plane_gs": lambda: run("plane_gs", level(lattice((2, 1, 1), (32, 32, 5))), "chaotic_block_gs",
                            (32, 32, 1)),
    "plane_gs_mixed": lambda: run("plane_gs_mixed", level([((9, 9, 9), (0, 0, 0)), ((16, 16, 16), (9, 0, 0))]),
                                  "chaotic_block_gs", (16, 16, 1)),
    "box_jacobi": lambda: run("box_jacobi", level([((20, 17, 11), (0, 0, 0))]), "block_jacobi", (8, 8, 8)),
    "box_gs": lambda: run("box_gs", level([((12, 10, 9), (0, 0, 0))]), "chaotic_block_gs", (4, 4, 4)),
    "ghosts_lattice_jacobi": lambda: run("ghosts_lattice_jacobi", level(lattice((2, 2, 2), (16, 12, 10))),
                                         "block_jacobi", (16, 1, 1)),
    # round 2: multi-sweep line GS (single patch, 4 steps in one launch)
    "gs_multisweep": lambda: run("gs_multisweep", level([((64, 10, 16), (0, 0, 0))]), "chaotic_block_gs",
                                 (64, 1, 1), steps=4),
    # DST tiles + one-launch chain (plane GS), DST tiles in Jacobi ('dst' mode)
    "plane_gs_dst_chain": lambda: run("plane_gs_dst_chain", level([((64, 48, 6), (0, 0, 0))]), "chaotic_block_gs",
                                      (64, 48, 1), steps=2),
    "plane_jacobi_dst": lambda: plane_dst_jacobi(),
    # persistent box GS (dependency flags)
    "box_gs_persistent": lambda: run("box_gs_persistent", level([((24, 16, 16), (0, 0, 0))]), "chaotic_block_gs",
                                     (8, 8, 8)),
    "api_primitives": lambda: api_primitives(),
    # box sweep: TMA staging + fragment-register passes (4^3 blocks in 8^3
    # regions), and the cp.async fallback of an odd-width patch
    "box_jacobi_4": lambda: run("box_jacobi_4", level([((24, 16, 13), (0, 0, 0))]), "block_jacobi", (4, 4, 4)),
    "box_jacobi_odd": lambda: run("box_jacobi_odd", level([((21, 16, 16), (0, 0, 0))]), "block_jacobi", (8, 8, 8)),
}


def plane_dst_jacobi():
    prev = ps.plane_solver("dst")
    try:
        run("plane_jacobi_dst", level([((40, 24, 5), (0, 0, 0))]), "block_jacobi", (40, 24, 1))
    finally:
        ps.plane_solver(prev)


def api_primitives():
    rng = np.random.default_rng(3)
    p = ps.Patch(ps.PatchDims(9, 7, 6))
    p.u.copy_(torch.from_numpy(rng.standard_normal(p.u.shape)))
    st = ps.Stencil7()
    ps.block_residual(st, p, ps.BlockRange((1, 2, 0), (8, 3, 6)))
    ps.apply_stencil(st, p, (4, 3, 2))
    m = rng.standard_normal((40, 40)) + 40 * np.eye(40)
    ps.matvec(m, rng.standard_normal(40))
    ps.block_update(rng.standard_normal(40), rng.standard_normal(40), m, 0.7)
    ps.invert_dense(m)
    torch.cuda.synchronize()
    print("api_primitives: ok", flush=True)
CHAOTIC = {
    "gs_pipe_chaotic": lambda: run("gs_pipe_chaotic", level(lattice((2, 1, 2), (64, 10, 9))), "chaotic_block_gs",
                                   (64, 1, 1), mode="chaotic"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chaotic", action="store_true")
    ap.add_argument("--only", nargs="*")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cases = dict(CASES)
    if a.chaotic:
        cases.update(CHAOTIC)
    for name, fn in cases.items():
        if a.only and name not in a.only:
            continue
        fn()


if __name__ == "__main__":
    main()
