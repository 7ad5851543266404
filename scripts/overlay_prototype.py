"""Numerics check for the bounded-overlay PSI design, host-only prototype.

A belief's PSI row is the initial row with k realised cells replaced.  The dense fast path builds
the fp32 CDF of softmax(eta * row) in column order; the overlay path would binary-search

    CDF(a) = s * initCDF(a) + sum_{a_j <= a} c_j,   s = exp(eta (LSE_init - LSE)),
    c_j = exp(eta psi_j - eta LSE) - exp(eta init_{a_j} - eta LSE)

with the shared initial CDF.  This script measures, in fp32 like the kernels, how often the two
pick different actions for the same uniform draw, and the largest CDF difference -- the tolerance
the fp32 sampler tests would have to accept.

    python scripts/overlay_prototype.py
"""
import numpy as np


def lse(row, eta):
    z = eta * row
    m = z.max()
    return (m + np.log(np.exp(z - m).sum())) / eta


def dense_cdf(row, eta):
    p = np.exp((eta * row - eta * lse(row, eta)).astype(np.float32))
    c = np.cumsum(p, dtype=np.float32)
    return c / c[-1]


def overlay_cdf(init, init_cdf, cells, vals, eta):
    row = init.copy()
    row[cells] = vals
    L, L0 = lse(row, eta), lse(init, eta)
    s = np.float32(np.exp(eta * (L0 - L)))
    corr = np.zeros(len(init), dtype=np.float32)
    corr[cells] = (np.exp(eta * vals - eta * L) - np.exp(eta * init[cells] - eta * L)).astype(np.float32)
    return s * init_cdf + np.cumsum(corr, dtype=np.float32)


def main():
    g = np.random.default_rng(0)
    eta = 2.0
    for A in (16, 256, 400):
        for k in (1, 2, 4):
            flips = draws = 0
            worst = 0.0
            for _ in range(400):
                init = g.normal(0.0, 0.5, size=A)
                init_cdf = dense_cdf(init, eta)
                cells = g.choice(A, size=k, replace=False)
                vals = init[cells] + g.normal(0.0, 3.0, size=k)
                row = init.copy()
                row[cells] = vals
                dc = dense_cdf(row, eta)
                oc = overlay_cdf(init, init_cdf, cells, vals, eta)
                worst = max(worst, float(np.abs(dc - oc).max()))
                u = g.random(256).astype(np.float32)
                a_dense = np.minimum(np.searchsorted(dc, u, side="right"), A - 1)
                a_over = np.minimum(np.searchsorted(oc, u, side="right"), A - 1)
                flips += int((a_dense != a_over).sum())
                draws += len(u)
            print(f"|A|={A:4d} k={k}: max |CDF_dense - CDF_overlay| = {worst:.2e}, "
                  f"action flips {flips}/{draws} = {flips / draws:.1e}")


if __name__ == "__main__":
    main()
