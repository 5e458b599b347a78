"""Near-minimax polynomial for atan(x) = x * P(x^2), |x| <= 0.4243 (y <= 0.18),
used by the fast SE3 log paths (lsh.cu kval_fast, particles.cu SVGD). Prints
the coefficients and the max relative error of the double-precision Horner
evaluation against mpmath."""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
Y = mp.mpf("0.18")


def g(y):
    if y == 0:
        return mp.mpf(1)
    r = mp.sqrt(y)
    return mp.atan(r) / r


def cheb_fit(n):
    # Chebyshev interpolation at n+1 nodes on [0, Y], then convert to monomials
    nodes = [Y / 2 * (1 - mp.cos(mp.pi * (k + mp.mpf(1) / 2) / (n + 1))) for k in range(n + 1)]
    vals = [g(x) for x in nodes]
    # solve Vandermonde in high precision
    A = mp.matrix([[x ** j for j in range(n + 1)] for x in nodes])
    c = mp.lu_solve(A, mp.matrix(vals))
    return [c[j] for j in range(n + 1)]


for n in (9, 10, 11, 12):
    c = cheb_fit(n)
    cf = [float(v) for v in c]
    xs = np.linspace(-0.4243, 0.4243, 200001)
    worst = 0.0
    for x in xs[::97]:
        y = x * x
        p = cf[-1]
        for a in reversed(cf[:-1]):
            p = p * y + a
        approx = x * p
        exact = mp.atan(mp.mpf(x))
        if exact != 0:
            worst = max(worst, abs((mp.mpf(approx) - exact) / exact))
    print(n, float(worst))
    if n == 11:
        print(",\n".join(repr(v) for v in cf))
