"""Fit the polynomial used by stk::fast_atan2 (paper_1912_04753_b200/csrc/stk_device.cuh).

atan(t) = t + t*s*R(s), s = t^2, |t| <= tan(pi/8).  R is fitted by least
squares on Chebyshev nodes in mpmath (60 digits) and its max error reported;
the coefficients are printed in the form pasted into the header.
"""
import mpmath as mp

mp.mp.dps = 60
TAN_PI_8 = mp.tan(mp.pi / 8)
SMAX = TAN_PI_8 ** 2


def R(s):
    if s == 0:
        return mp.mpf(-1) / 3
    t = mp.sqrt(s)
    return (mp.atan(t) - t) / (t * s)


def fit(deg, nodes=400):
    xs = [SMAX * (1 - mp.cos(mp.pi * (k + mp.mpf(1) / 2) / nodes)) / 2 for k in range(nodes)]
    A = mp.matrix(nodes, deg + 1)
    b = mp.matrix(nodes, 1)
    for i, x in enumerate(xs):
        for j in range(deg + 1):
            A[i, j] = x ** j
        b[i] = R(x)
    coef = mp.lu_solve(A.T * A, A.T * b)
    return [coef[j] for j in range(deg + 1)]


def max_err(coef, samples=3000):
    worst = 0
    for k in range(samples + 1):
        t = TAN_PI_8 * k / samples
        s = t * t
        r = sum(c * s ** j for j, c in enumerate(coef))
        approx = t + t * s * r
        exact = mp.atan(t)
        if t > 0:
            worst = max(worst, abs(approx - exact) / exact)
    return worst


for deg in (9, 10, 11, 12):
    c = fit(deg)
    print(deg, mp.nstr(max_err(c), 5))
c = fit(11)
print("coefficients (R(s) = sum c_j s^j):")
for j, v in enumerate(c):
    print(f"  {mp.nstr(v, 20)},")
