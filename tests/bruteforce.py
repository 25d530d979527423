"""O0: pure-Python brute force of one IFCM step (test infrastructure).

Independent of oracle/pifcm_oracle.c: it loops over ALL voxel pairs (i, k)
and decides membership of the neighbourhood with the literal Eq. 9 test
 with L = 3, i.e. 0 < dX^2 + dY^2 + dZ^2 < 2^(L-1) = 4, and uses
Eq. 8's q squared per Eq. 7 (LITERAL) or unsquared
(SQEUCLID).  Single shell (v = 1, W_1 = 1 by Eq. 10).  Only for tiny inputs
(O(N^2) Python loops).
"""
from __future__ import annotations

import math


def ifcm_step_bruteforce(x, U, c, lam, xi, m=2.0, q_mode=0):
    """x: nested lists/array [nz][ny][nx]; U: [N][C]; c: [C]."""
    nz = len(x)
    ny = len(x[0])
    nx = len(x[0][0])
    coords = [(X, Y, Z) for Z in range(nz) for Y in range(ny) for X in range(nx)]
    xs = [float(x[Z][Y][X]) for (X, Y, Z) in coords]
    N = len(coords)
    C = len(c)
    U_new = [[0.0] * C for _ in range(N)]
    num = [0.0] * C
    den = [0.0] * C
    J = 0.0
    maxdu = 0.0
    L = 3
    for i in range(N):
        Xi, Yi, Zi = coords[i]
        Gsum = 0.0
        Qsum = 0.0
        Hn = [0.0] * C
        Fn = [0.0] * C
        for k in range(N):
            Xk, Yk, Zk = coords[k]
            dist2 = (Xi - Xk) ** 2 + (Yi - Yk) ** 2 + (Zi - Zk) ** 2
            if not (0 < dist2 < 2 ** (L - 1)):
                continue
            g = abs(xs[i] - xs[k])
            q = dist2
            q2 = q * q if q_mode == 0 else q
            Gsum += g
            Qsum += q2
            for j in range(C):
                Hn[j] += float(U[k][j]) * g
                Fn[j] += float(U[k][j]) ** 2 * q2
        d2 = []
        for j in range(C):
            H = Hn[j] / Gsum if Gsum > 0 else 0.0
            F = Fn[j] / Qsum if Qsum > 0 else 0.0
            a = max(1.0 - lam * H - xi * F, 1e-9)
            d2.append((xs[i] - float(c[j])) ** 2 * a)
        zero = [j for j in range(C) if d2[j] == 0.0]
        for j in range(C):
            if zero:
                u = 1.0 if j == zero[0] else 0.0
            else:
                u = 1.0 / sum((d2[j] / d2[k]) ** (1.0 / (m - 1.0)) for k in range(C))
            U_new[i][j] = u
            um = u ** m
            num[j] += um * xs[i]
            den[j] += um
            J += um * d2[j]
            maxdu = max(maxdu, abs(u - float(U[i][j])))
    c_new = [num[j] / den[j] if den[j] >= 1e-12 else float(c[j]) for j in range(C)]
    return U_new, c_new, J, maxdu


def neighbour_count_bruteforce(nx, ny, nz, X, Y, Z):
    """Number of voxels satisfying Eq. 9 (L = 3) around (X, Y, Z)."""
    n = 0
    for Zk in range(nz):
        for Yk in range(ny):
            for Xk in range(nx):
                d = (X - Xk) ** 2 + (Y - Yk) ** 2 + (Z - Zk) ** 2
                if 0 < d < 4:
                    n += 1
    return n


def qsum_bruteforce(nx, ny, nz, X, Y, Z, q_mode=0):
    s = 0
    for Zk in range(nz):
        for Yk in range(ny):
            for Xk in range(nx):
                d = (X - Xk) ** 2 + (Y - Yk) ** 2 + (Z - Zk) ** 2
                if 0 < d < 4:
                    s += d * d if q_mode == 0 else d
    return s


def isclose(a, b, tol):
    return math.isclose(a, b, rel_tol=0.0, abs_tol=tol)


def ifcm_step_bruteforce_shells(x, U, c, lam, xi, v, h, m=2.0, q_mode=0):
    """One IFCM step with v Chebyshev shells (reading R2 of Eq. 9 for v >= 2)
    weighted by Eq. 10: W_r = e^{-r/h} / sum_{s=1..v} e^{-s/h};
    every shell is normalised on its own (its own G and Qs), a shell whose
    g's are all zero contributes 0 (R3).  Pairwise over all voxel pairs."""
    nz, ny, nx = len(x), len(x[0]), len(x[0][0])
    coords = [(X, Y, Z) for Z in range(nz) for Y in range(ny) for X in range(nx)]
    xs = [float(x[Z][Y][X]) for (X, Y, Z) in coords]
    N, C = len(coords), len(c)
    den_w = sum(math.exp(-s / h) for s in range(1, v + 1))
    W = [math.exp(-r / h) / den_w for r in range(1, v + 1)]
    U_new = [[0.0] * C for _ in range(N)]
    num, den = [0.0] * C, [0.0] * C
    J, maxdu = 0.0, 0.0
    for i in range(N):
        Xi, Yi, Zi = coords[i]
        G = [0.0] * v
        Q = [0.0] * v
        Hn = [[0.0] * C for _ in range(v)]
        Fn = [[0.0] * C for _ in range(v)]
        for k in range(N):
            Xk, Yk, Zk = coords[k]
            r = max(abs(Xi - Xk), abs(Yi - Yk), abs(Zi - Zk))
            if r == 0 or r > v:
                continue
            q = (Xi - Xk) ** 2 + (Yi - Yk) ** 2 + (Zi - Zk) ** 2
            q2 = q * q if q_mode == 0 else q
            g = abs(xs[i] - xs[k])
            G[r - 1] += g
            Q[r - 1] += q2
            for j in range(C):
                Hn[r - 1][j] += float(U[k][j]) * g
                Fn[r - 1][j] += float(U[k][j]) ** 2 * q2
        d2 = []
        for j in range(C):
            H = sum(W[s] * Hn[s][j] / G[s] for s in range(v) if G[s] > 0)
            F = sum(W[s] * Fn[s][j] / Q[s] for s in range(v) if Q[s] > 0)
            a = max(1.0 - lam * H - xi * F, 1e-9)
            d2.append((xs[i] - float(c[j])) ** 2 * a)
        zero = [j for j in range(C) if d2[j] == 0.0]
        for j in range(C):
            if zero:
                u = 1.0 if j == zero[0] else 0.0
            else:
                u = 1.0 / sum((d2[j] / d2[k]) ** (1.0 / (m - 1.0)) for k in range(C))
            U_new[i][j] = u
            um = u ** m
            num[j] += um * xs[i]
            den[j] += um
            J += um * d2[j]
            maxdu = max(maxdu, abs(u - float(U[i][j])))
    c_new = [num[j] / den[j] if den[j] >= 1e-12 else float(c[j]) for j in range(C)]
    return U_new, c_new, J, maxdu
