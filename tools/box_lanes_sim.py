"""Lane-order check for the fragment-register DMMA passes of box_sweep_t (psm_box.cu).

Simulates the six m8n8k4 passes of one interior 8^3 region lane by lane: the
residual loaded straight into the x-pass B fragments in line order box_jx,
the three two-shuffle register exchanges (x -> y, z -> z', y' -> x'), the two
work-cube transposes (y -> z, z' -> y') in line order box_ip, and the relax
read of the halo.  It compares the result with the separable transform
applied directly and checks that every shared-memory access is bank-conflict
free under the half-warp model of 8-byte accesses (16 distinct 8-byte banks
per half warp).  Pure numpy; run: python tools/box_lanes_sim.py
"""
import numpy as np

RS, RP = 12, 100  # work cube: row and plane strides (kRs, kRp)
HS, HP = 10, 100  # staged halo box: row and plane strides (kHs, kHp)
FS = 10           # staged f: row stride


def jx(n):  # x pass: line n -> row j
    return 2 * (n & 3) + (n >> 2)


def ip(n):  # y pass / z' pass: line n -> column i
    return (n >> 1) + 4 * (n & 1)


def dmma(A, bfrag):
    """m8n8k4 over a warp: bfrag[lane][ks] is B[4 ks + lane%4][lane/4];
    returns D fragments d[lane][e] = D[lane/4][2 (lane%4) + e]."""
    B = np.zeros((8, 8))
    for lane in range(32):
        for ks in range(2):
            B[4 * ks + (lane & 3)][lane >> 2] = bfrag[lane][ks]
    D = A @ B
    return [[D[lane >> 2][2 * (lane & 3) + e] for e in range(2)] for lane in range(32)]


def simulate(seed=0):
    """Returns (max error relative to max |direct transform|, list of bank conflicts)."""
    rng = np.random.default_rng(seed)
    M = [rng.standard_normal((8, 8)) for _ in range(6)]
    scale = rng.standard_normal((8, 8, 8))  # 1/lambda [k][j][i]
    R = rng.standard_normal((8, 8, 8))      # residual [k][j][i]
    X = np.einsum("ip,kjp->kji", M[0], R)
    X = np.einsum("jp,kpi->kji", M[1], X)
    X = np.einsum("kp,pji->kji", M[2], X) * scale
    X = np.einsum("kp,pji->kji", M[3], X)
    X = np.einsum("jp,kpi->kji", M[4], X)
    ref = np.einsum("ip,kjp->kji", M[5], X)

    issues = []

    def check(name, addrs):
        for h in range(2):
            banks = [addrs[lane] % 16 for lane in range(16 * h, 16 * h + 16)]
            if len(set(banks)) != 16:
                issues.append((name, h, sorted(banks)))

    wc = np.full(8 * RP, np.nan)
    out = np.zeros((8, 8, 8))
    dz2_of = {}
    # residual -> x -> (shuffles) -> y -> cube, warp w owns planes k = 2w, 2w+1
    for w in range(4):
        for tt in range(2):
            k = 2 * w + tt
            bx = [[R[k][jx(l >> 2)][4 * ks + (l & 3)] for ks in range(2)] for l in range(32)]
            for ks in range(2):
                for off in (0, -1, 1, -HS, HS, -HP, HP):
                    check("residual halo", [(k + 1) * HP + (jx(l >> 2) + 1) * HS + 4 * ks + (l & 3) + 1 + off
                                            for l in range(32)])
                check("residual f", [(k * 8 + jx(l >> 2)) * FS + 4 * ks + (l & 3) for l in range(32)])
            dx = dmma(M[0], bx)
            by = [[None, None] for _ in range(32)]
            for sh in range(2):  # sender element d[c & 1], then the other
                send = [dx[l][(l & 1) ^ sh] for l in range(32)]
                for l in range(32):
                    r, c = l >> 2, l & 3
                    src = ip(r) * 4 + ([0, 2, 1, 3] if sh == 0 else [1, 3, 0, 2])[c]
                    by[l][(c >> 1) if sh == 0 else 1 - (c >> 1)] = send[src]
            dy = dmma(M[1], by)
            for e in range(2):
                ad = [k * RP + (l >> 2) * RS + ip(2 * (l & 3) + e) for l in range(32)]
                check("y store", ad)
                for l in range(32):
                    wc[ad[l]] = dy[l][e]
    # z -> (shuffles) -> z', warp w owns planes j = 2w, 2w+1
    for w in range(4):
        for tt in range(2):
            j = 2 * w + tt
            bz = [[None, None] for _ in range(32)]
            for ks in range(2):
                ad = [(4 * ks + (l & 3)) * RP + j * RS + (l >> 2) for l in range(32)]
                check("z load", ad)
                for l in range(32):
                    bz[l][ks] = wc[ad[l]]
            dz = dmma(M[2], bz)
            for l in range(32):
                for e in range(2):
                    dz[l][e] *= scale[l >> 2][j][2 * (l & 3) + e]
            bz2 = [[None, None] for _ in range(32)]
            for sh in range(2):  # sender element d[lane/4 >= 4], then the other
                send = [dz[l][int((l >> 2) >= 4) ^ sh] for l in range(32)]
                for l in range(32):
                    r, c = l >> 2, l & 3
                    e = ip(r) & 1
                    rs = (4 + c if e else c) if sh == 0 else (c if e else 4 + c)
                    bz2[l][e if sh == 0 else 1 - e] = send[rs * 4 + (ip(r) >> 1)]
            dz2_of[(w, tt)] = dmma(M[3], bz2)
    for w in range(4):
        for tt in range(2):
            j = 2 * w + tt
            for e in range(2):
                ad = [(l >> 2) * RP + j * RS + ip(2 * (l & 3) + e) for l in range(32)]
                check("z' store", ad)
                for l in range(32):
                    wc[ad[l]] = dz2_of[(w, tt)][l][e]
    # y' -> (shuffles) -> x' -> relax, warp w owns planes k = 2w, 2w+1
    for w in range(4):
        for tt in range(2):
            k = 2 * w + tt
            by2 = [[None, None] for _ in range(32)]
            for ks in range(2):
                ad = [k * RP + (4 * ks + (l & 3)) * RS + (l >> 2) for l in range(32)]
                check("y' load", ad)
                for l in range(32):
                    by2[l][ks] = wc[ad[l]]
            dy2 = dmma(M[4], by2)
            bx2 = [[None, None] for _ in range(32)]
            for sh in range(2):  # within the quad: sender element d[c >> 1], then the other
                send = [dy2[l][((l & 3) >> 1) ^ sh] for l in range(32)]
                for l in range(32):
                    r, c = l >> 2, l & 3
                    bx2[l][(c & 1) ^ sh] = send[r * 4 + (c >> 1) + 2 * ((c & 1) ^ sh)]
            dx2 = dmma(M[5], bx2)
            for e in range(2):
                check("relax halo", [(k + 1) * HP + (2 * (l & 3) + e + 1) * HS + (l >> 2) + 1 for l in range(32)])
                for l in range(32):
                    out[k][2 * (l & 3) + e][l >> 2] = dx2[l][e]
    return float(np.abs(out - ref).max() / np.abs(ref).max()), issues


if __name__ == "__main__":
    err, issues = simulate()
    print("max rel err", err)
    print("bank conflicts", len(issues), issues[:5])
