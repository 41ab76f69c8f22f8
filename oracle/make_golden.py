"""Generate tests/golden/*.npz by running the REFERENCE package itself.

TEST INFRASTRUCTURE ONLY.  Run in the dev container, where the read-only
reference lives at /root/reference (it does not exist on the GPU box, so the
outputs are committed as small fixtures):

    python oracle/make_golden.py [--only-box]

Every case builds its inputs with seeded numpy generators, runs
``patchsmooth.smooth`` (``/root/reference/pkg/src/patchsmooth/smoother.py:197``)
and stores inputs, final interiors (or samples of them for the larger cases)
and the residual history.  Case names encode the configuration.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    sys.path.insert(0, REF)
    import patchsmooth  # noqa: E402

    return patchsmooth


def _save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path)} bytes")


def _stencil(ps, kind):
    if kind == "default":
        return ps.Stencil7()
    if kind == "aniso_line":  # asymmetric faces: only line blocks support these
        return ps.Stencil7(center=7.5, faces=(-1.2, -0.8, -1.1, -0.9, -1.0, -1.3))
    if kind == "aniso_plane":  # symmetric in x, asymmetric in y/z
        return ps.Stencil7(center=7.0, faces=(-1.5, -1.5, -0.7, -1.2, -1.0, -1.1))
    raise ValueError(kind)


def random_patch_case(ps, name, shape, block, scheme, steps, omega=None, seed=11,
                      stencil="default"):
    rng = np.random.default_rng(seed)
    p = ps.Patch(ps.PatchDims(*shape))
    u0 = rng.standard_normal(shape)
    f = rng.standard_normal(shape)
    p.u[1:-1, 1:-1, 1:-1] = u0
    p.f[:] = f
    level = ps.Level([p])
    st = _stencil(ps, stencil)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, omega=omega, steps=steps, stencil=st)
    _, hist = ps.smooth(level, cfg, ps.InverseCache())
    _save(name, shape=np.array(shape), block=np.array(block), scheme=np.array(scheme),
          omega=np.array(cfg.omega), steps=np.array(steps), center=np.array(st.center),
          faces=np.array(st.faces), u0=u0, f=f, u_final=np.array(p.u), history=np.array(hist))


def lattice(ps, counts, size):
    patches = []
    for c in range(counts[2]):
        for b in range(counts[1]):
            for a in range(counts[0]):
                patches.append(ps.Patch(ps.PatchDims(*size), origin=(a * size[0], b * size[1], c * size[2])))
    return ps.Level(patches)


def multipatch_case(ps, name, counts, size, block, scheme, steps, seed=5):
    level = lattice(ps, counts, size)
    rng = np.random.default_rng(seed)
    u0, f0 = [], []
    for p in level.patches:
        a = rng.standard_normal(size)
        b = rng.standard_normal(size)
        p.u[1:-1, 1:-1, 1:-1] = a
        p.f[:] = b
        u0.append(a)
        f0.append(b)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=steps)
    _, hist = ps.smooth(level, cfg, ps.InverseCache())
    adj = np.array([[c.src, c.dst, *c.src_lo, *c.dst_lo, *c.extent] for c in level.adjacency])
    _save(name, counts=np.array(counts), size=np.array(size), block=np.array(block),
          scheme=np.array(scheme), omega=np.array(cfg.omega), steps=np.array(steps),
          u0=np.stack(u0), f=np.stack(f0), u_final=np.stack([np.array(p.u) for p in level.patches]),
          history=np.array(hist), adjacency=adj)


def zsplit_case(ps, name, shape, parts, block, scheme, steps, seed=8):
    """One patch cut into `parts` z-slabs (the multi-GPU decomposition)."""
    nx, ny, nz = shape
    dz = nz // parts
    patches = [ps.Patch(ps.PatchDims(nx, ny, dz), origin=(0, 0, g * dz)) for g in range(parts)]
    level = ps.Level(patches)
    rng = np.random.default_rng(seed)
    u0 = rng.standard_normal(shape)
    f = rng.standard_normal(shape)
    for g, p in enumerate(patches):
        p.u[1:-1, 1:-1, 1:-1] = u0[:, :, g * dz:(g + 1) * dz]
        p.f[:] = f[:, :, g * dz:(g + 1) * dz]
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=steps)
    _, hist = ps.smooth(level, cfg, ps.InverseCache())
    final = np.concatenate([np.array(p.interior) for p in patches], axis=2)
    _save(name, shape=np.array(shape), parts=np.array(parts), block=np.array(block),
          scheme=np.array(scheme), omega=np.array(cfg.omega), steps=np.array(steps),
          u0=u0, f=f, interior_final=final, history=np.array(hist))


def seeded_case(ps, name, shape, block, scheme, steps, sample_planes=(0,)):
    """bench.seed_initial_guess(level, 42), f = 0: the CLI's own inputs."""
    level = ps.build_level([shape])
    ps.seed_initial_guess(level, 42)
    cfg = ps.SmootherConfig(scheme=scheme, block_dims=block, steps=steps)
    t0 = time.perf_counter()
    _, hist = ps.smooth(level, cfg, ps.InverseCache())
    print(f"  {name}: smooth took {time.perf_counter() - t0:.1f} s")
    inter = np.array(level.patches[0].interior)
    _save(name, shape=np.array(shape), block=np.array(block), scheme=np.array(scheme),
          omega=np.array(cfg.omega), steps=np.array(steps), history=np.array(hist),
          planes=np.array(sample_planes), plane_values=np.stack([inter[:, :, k] for k in sample_planes]),
          checksum=np.array([inter.sum(), np.square(inter).sum()]))


def host_logic_case(ps):
    """Adjacency and decomposition answers for host-side logic tests."""
    out = {}
    lv = ps.build_level([(4, 3, 2), (2, 3, 2), (3, 3, 2)])
    out["build_level_adj"] = np.array([[c.src, c.dst, *c.src_lo, *c.dst_lo, *c.extent] for c in lv.adjacency])
    # partial-face abutment: a 4x4x4 patch beside two 4x2x4 patches
    lv2 = ps.Level([ps.Patch(ps.PatchDims(4, 4, 4)),
                    ps.Patch(ps.PatchDims(4, 2, 4), origin=(4, 0, 0)),
                    ps.Patch(ps.PatchDims(4, 2, 4), origin=(4, 2, 0)),
                    ps.Patch(ps.PatchDims(3, 4, 2), origin=(1, 0, 4))])
    out["partial_adj"] = np.array([[c.src, c.dst, *c.src_lo, *c.dst_lo, *c.extent] for c in lv2.adjacency])
    lv3 = lattice(ps, (3, 2, 2), (3, 2, 4))
    out["lattice_adj"] = np.array([[c.src, c.dst, *c.src_lo, *c.dst_lo, *c.extent] for c in lv3.adjacency])
    # ghost refresh of a random multi-patch level, bitwise (all padded cells)
    rng = np.random.default_rng(77)
    for p in lv2.patches:
        p.u[...] = rng.standard_normal(p.u.shape)
    before = [np.array(p.u) for p in lv2.patches]
    lv2.refresh_ghosts()
    for i, (b, p) in enumerate(zip(before, lv2.patches)):
        out[f"refresh_before_{i}"] = b
        out[f"refresh_after_{i}"] = np.array(p.u)
    nrm = ps.residual_norm(lv2, ps.Stencil7())
    fs = []
    for p in lv2.patches:
        p.f[:] = rng.standard_normal(p.f.shape)
        fs.append(np.array(p.f))
    out["norm_f_zero"] = np.array(nrm)
    out["norm_with_f"] = np.array(ps.residual_norm(lv2, ps.Stencil7()))
    for i, f in enumerate(fs):
        out[f"norm_f_{i}"] = f
    _save("host_logic", **out)


def box_cases(ps):
    """Box blocks (the paper's cubic blocks, DEFAULT_BLOCK_SIZES), including
    blocks truncated at patch edges and x-segments shorter than the line."""
    for scheme in ("block_jacobi", "chaotic_block_gs"):
        tag = "jac" if scheme == "block_jacobi" else "gs"
        random_patch_case(ps, f"box_{tag}_16x12x10_b4x4x4", (16, 12, 10), (4, 4, 4), scheme, 2, seed=21)
        random_patch_case(ps, f"box_{tag}_8x8x8_b2x2x2", (8, 8, 8), (2, 2, 2), scheme, 3, seed=22)
        random_patch_case(ps, f"box_{tag}_17x9x11_b8x8x8", (17, 9, 11), (8, 8, 8), scheme, 2, seed=23)
        random_patch_case(ps, f"box_{tag}_aniso_12x8x6_b4x2x2", (12, 8, 6), (4, 2, 2), scheme, 2, seed=24,
                          stencil="aniso_line")
        random_patch_case(ps, f"box_{tag}_12x10x8_b8x1x1", (12, 10, 8), (8, 1, 1), scheme, 2, seed=25)
        multipatch_case(ps, f"multi_box_{tag}_2x2x2_of_8", (2, 2, 2), (8, 8, 8), (4, 4, 4), scheme, 2)
    random_patch_case(ps, "box_jac_w06_10x10x10_b4x4x4", (10, 10, 10), (4, 4, 4), "block_jacobi", 2, omega=0.6,
                      seed=26)
    random_patch_case(ps, "box_gs_9x9x9_b3x3x3", (9, 9, 9), (3, 3, 3), "chaotic_block_gs", 3, seed=27)


CLI_CASES = {
    "cli_converge_default_12": ["converge", "--patch-size", "12x12x12", "--steps", "4"],
    "cli_converge_gs_10x9x8": ["converge", "--patch-size", "10x9x8", "--scheme", "chaotic-gs", "--steps", "3",
                               "--block-size", "4x4x2"],
    "cli_smooth_box_16_n2": ["smooth", "--patch-size", "16x16x16", "--num-patches", "2", "--steps", "3"],
    "cli_smooth_lines_mixed": ["smooth", "--patch-size", "24x8x8", "--patch-size", "16x8x8", "--block-size",
                               "24x1x1", "--scheme", "chaotic-gs", "--steps", "2"],
    "cli_smooth_plane_w06": ["smooth", "--patch-size", "16x12x6", "--block-size", "16x12x1", "--omega", "0.6",
                             "--steps", "3"],
}


def cli_cases():
    """The reference CLI's own CSV output (cli.py:319-358) for small cases."""
    sys.path.insert(0, REF)
    import io
    from contextlib import redirect_stdout

    from patchsmooth import cli

    for name, argv in CLI_CASES.items():
        buf = io.StringIO()
        with redirect_stdout(buf):
            rc = cli.main(argv)
        assert rc == 0, (name, rc)
        path = os.path.join(OUT, name + ".csv")
        with open(path, "w", newline="") as fh:
            fh.write(buf.getvalue())
        with open(path + ".args", "w") as fh:
            fh.write(" ".join(argv) + "\n")
        print(f"wrote {name}: {os.path.getsize(path)} bytes")


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--only-cli" in sys.argv:
        cli_cases()
        return
    if "--only-box" in sys.argv:
        box_cases(_ref())
        return
    ps = _ref()
    t0 = time.perf_counter()
    # single patch, random u and f
    for scheme in ("block_jacobi", "chaotic_block_gs"):
        tag = "jac" if scheme == "block_jacobi" else "gs"
        random_patch_case(ps, f"line_{tag}_12x10x8", (12, 10, 8), (12, 1, 1), scheme, 3)
        random_patch_case(ps, f"line_{tag}_32x6x5", (32, 6, 5), (64, 1, 1), scheme, 2)
        random_patch_case(ps, f"line_{tag}_64x8x7", (64, 8, 7), (64, 1, 1), scheme, 3, seed=12)
        random_patch_case(ps, f"line_{tag}_96x5x4", (96, 5, 4), (96, 1, 1), scheme, 2, seed=13)
        random_patch_case(ps, f"line_{tag}_aniso_10x6x5", (10, 6, 5), (10, 1, 1), scheme, 3, stencil="aniso_line")
        random_patch_case(ps, f"line_{tag}_aniso_64x4x3", (64, 4, 3), (64, 1, 1), scheme, 2, stencil="aniso_line")
        random_patch_case(ps, f"plane_{tag}_8x6x5", (8, 6, 5), (8, 6, 1), scheme, 3)
        random_patch_case(ps, f"plane_{tag}_16x16x6", (16, 16, 6), (16, 16, 1), scheme, 2)
        random_patch_case(ps, f"plane_{tag}_aniso_8x7x4", (8, 7, 4), (8, 7, 1), scheme, 2, stencil="aniso_plane")
        random_patch_case(ps, f"line_{tag}_odd_7x5x3", (7, 5, 3), (9, 1, 1), scheme, 2)
        random_patch_case(ps, f"plane_{tag}_odd_5x3x2", (5, 3, 2), (5, 4, 1), scheme, 2)
        random_patch_case(ps, f"line_{tag}_1x1x1", (1, 1, 1), (1, 1, 1), scheme, 2)
    random_patch_case(ps, "line_gs_w07_12x10x8", (12, 10, 8), (12, 1, 1), "chaotic_block_gs", 2, omega=0.7)
    random_patch_case(ps, "line_jac_w05_12x10x8", (12, 10, 8), (12, 1, 1), "block_jacobi", 2, omega=0.5)
    random_patch_case(ps, "plane_gs_w07_8x6x5", (8, 6, 5), (8, 6, 1), "chaotic_block_gs", 2, omega=0.7)
    # multi-patch lattices (AMR-style, C4 in miniature)
    for scheme in ("block_jacobi", "chaotic_block_gs"):
        tag = "jac" if scheme == "block_jacobi" else "gs"
        multipatch_case(ps, f"multi_line_{tag}_2x2x2_of_8", (2, 2, 2), (8, 8, 8), (8, 1, 1), scheme, 3)
        multipatch_case(ps, f"multi_plane_{tag}_2x2x2_of_8", (2, 2, 2), (8, 8, 8), (8, 8, 1), scheme, 2)
        multipatch_case(ps, f"multi_line_{tag}_3x1x2_of_32x4x3", (3, 1, 2), (32, 4, 3), (32, 1, 1), scheme, 2)
        zsplit_case(ps, f"zsplit_line_{tag}_32x8x8_in4", (32, 8, 8), 4, (32, 1, 1), scheme, 3)
    zsplit_case(ps, "zsplit_plane_jac_8x8x8_in2", (8, 8, 8), 2, (8, 8, 1), "block_jacobi", 2)
    box_cases(ps)
    cli_cases()
    host_logic_case(ps)
    # the CLI's own inputs (seed 42, f = 0) -- SURVEY section 8c golden histories
    seeded_case(ps, "seeded_line_jac_64", (64, 64, 64), (64, 1, 1), "block_jacobi", 10, (0, 31, 63))
    seeded_case(ps, "seeded_line_gs_32", (32, 32, 32), (32, 1, 1), "chaotic_block_gs", 8, (0, 15))
    seeded_case(ps, "seeded_plane_jac_32", (32, 32, 32), (32, 32, 1), "block_jacobi", 3, (0, 15))
    print(f"total {time.perf_counter() - t0:.1f} s")


if __name__ == "__main__":
    main()
