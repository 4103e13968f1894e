"""Independent LP oracle for the strategy optimizer (scipy HiGHS).

TEST INFRASTRUCTURE ONLY. Restates DeDLOC's Eq. 5 in the
compact form of /root/reference/proj/src/strategy.cpp:193-295 in consistent
units (flows in Gbit/s, payload in Gbit), with every computing peer's duty
cycle pinned to 1 (the 0/1 restriction of strategy.cpp:329-404 selects "all
on" for every reference fixture), then stage C (max sum_i min_j g_ij,
strategy.cpp:422-441) and stage D (min total flow, :443-451), and returns
(xi, fractions). Pinned by the reference's frozen goldens
(/root/reference/proj/tests/cpp/test_strategy.cpp:189,200,213-220)."""
from __future__ import annotations

import numpy as np
from scipy.optimize import linprog


def solve(spec: dict, method: str = "highs-ds"):
    peers = spec["peers"]
    n = len(peers)
    B = spec.get("batch_size", 1.0)
    P = spec["param_count"] * spec.get("bits_per_param", 32.0) / 1e9  # Gbit
    d = np.array([p["download_mbps"] / 1e3 for p in peers])  # Gbit/s
    u = np.array([p["upload_mbps"] / 1e3 for p in peers])
    s = np.array([p.get("samples_per_sec", 0.0) for p in peers])
    can = np.array([p.get("can_compute", True) for p in peers])
    client = np.array([p.get("client_mode", False) for p in peers])
    comp = can & (s > 0)
    recip = can & ~client
    # variables: a (n*n), g (n*n), xi, M (n)
    A_, G_, XI, M_ = 0, n * n, 2 * n * n, 2 * n * n + 1
    nv = 2 * n * n + 1 + n
    a = lambda i, j: A_ + i * n + j  # noqa: E731
    g = lambda i, j: G_ + i * n + j  # noqa: E731
    ub = np.full(nv, np.inf)
    for i in range(n):
        for j in range(n):
            if j != i and client[j]:
                ub[a(i, j)] = ub[g(i, j)] = 0.0
            if not comp[i]:
                ub[a(i, j)] = 0.0
            if not recip[j]:
                ub[g(i, j)] = 0.0
    rows, rhs = [], []

    def row(terms, b):
        r = np.zeros(nv)
        for k, c in terms:
            r[k] += c
        rows.append(r)
        rhs.append(b)

    row([(XI, 1.0)], s[comp].sum() / B)  # c pinned to 1
    for i in np.flatnonzero(recip):
        row([(XI, P)] + [(g(j, i), -1.0) for j in range(n)], 0.0)
    if recip.any():
        for i in range(n):
            for j in np.flatnonzero(recip):
                row([(g(i, j), 1.0), (M_ + i, -1.0)], 0.0)
            for k in np.flatnonzero(comp):
                row([(M_ + i, 1.0), (a(k, i), -1.0)], 0.0)  # d_i (1 - c_k) = 0
    for i in range(n):
        row([(a(j, i), 1.0) for j in range(n) if j != i] + [(g(j, i), 1.0) for j in range(n) if j != i], d[i])
        row([(a(i, j), 1.0) for j in range(n) if j != i] + [(g(i, j), 1.0) for j in range(n) if j != i], u[i])
    A = np.array(rows)
    b = np.array(rhs)
    bounds = list(zip(np.zeros(nv), ub))
    c = np.zeros(nv)
    c[XI] = -1.0
    r = linprog(c, A_ub=A, b_ub=b, bounds=bounds, method=method)
    assert r.status == 0, r.message
    xi = r.x[XI]
    # stage C: f_i <= g_ij (j in R), maximize sum f
    nf = n
    A2 = np.hstack([A, np.zeros((A.shape[0], nf))])
    extra = []
    for i in range(n):
        for j in np.flatnonzero(recip):
            rr = np.zeros(nv + nf)
            rr[nv + i] = 1.0
            rr[g(i, j)] = -1.0
            extra.append(rr)
    A2 = np.vstack([A2] + extra) if extra else A2
    b2 = np.concatenate([b, np.zeros(len(extra))])
    bounds2 = bounds[:]
    bounds2[XI] = (xi * (1 - 1e-12), xi)
    bounds2 += [(0, np.inf)] * nf
    c2 = np.zeros(nv + nf)
    c2[nv:] = -1.0
    r2 = linprog(c2, A_ub=A2, b_ub=b2, bounds=bounds2, method=method)
    assert r2.status == 0, r2.message
    f = np.clip(r2.x[nv:], 0, None)
    fr = f / f.sum() if f.sum() > 0 else f
    return xi * 1.0, fr.tolist()
