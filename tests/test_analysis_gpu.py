"""The device convergence study (analysis.run_convergence_study)
against spectral radii computed by the reference's own dense power
iteration (spectral_radius_oracle; values pinned in the reference's
test_analysis.py:26-43 and SURVEY 8c): the measured asymptotic factor over
a window past the transient agrees with rho."""

import pytest

import paper_1208_1975_b200 as ps

pytestmark = pytest.mark.gpu

# (patch, block, scheme) -> rho from the reference (8^3 patch, default omega)
RHO = {
    ((8, 8, 8), (2, 2, 2), "block_jacobi"): 0.887449423164,
    ((8, 8, 8), (4, 4, 4), "block_jacobi"): 0.819677353342,
    ((8, 8, 8), (8, 4, 4), "block_jacobi"): 0.762357349716,
    ((8, 8, 8), (4, 2, 2), "chaotic_block_gs"): 0.697924729351,
    ((8, 8, 8), (8, 1, 1), "block_jacobi"): 0.911618881,
    ((8, 8, 8), (8, 1, 1), "chaotic_block_gs"): 0.788402184,
    ((8, 8, 8), (8, 8, 1), "block_jacobi"): 0.839037027,
    ((12, 12, 12), (12, 1, 1), "block_jacobi"): 0.959740910,
    ((12, 12, 12), (12, 12, 1), "chaotic_block_gs"): 0.815477956,
}


@pytest.mark.parametrize("key", sorted(RHO, key=str))
def test_measured_factor_matches_reference_spectral_radius(key):
    dims, block, scheme = key
    rho = RHO[key]
    import math

    # window well past the transient, ending before the rounding floor (1e-12)
    end = int(math.log(1e-11) / math.log(rho))
    start, length = end // 2, end - end // 2
    rep, = ps.run_convergence_study(ps.PatchDims(*dims), block_sizes=[block], schemes=[scheme], steps=end + 1,
                                    window=(start, length))
    assert rep.asymptotic_factor == pytest.approx(rho, rel=0.01), (rep.asymptotic_factor, rho)
