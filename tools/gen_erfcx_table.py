"""Generate the piecewise-polynomial erfcx(x) = exp(x^2) erfc(x) table used
by the real-space kernel: 12 intervals of width 0.5 on [0, 6), degree 12 in
t = 4x - (4a+1) in [-1, 1] per interval (a = interval start).  Chebyshev
interpolation at 40-digit precision, converted to monomials, rounded to
double.  Prints the C initialiser and the max relative error (double
Horner) against mpmath."""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
W, NI, DEG = 0.5, 12, 12


def erfcx(x):
    x = mp.mpf(x)
    return mp.exp(x * x) * mp.erfc(x)


def fit(a):
    n = DEG + 1
    ts = [mp.cos(mp.pi * (k + mp.mpf(1) / 2) / n) for k in range(n)]
    ys = [erfcx(a + (t + 1) * W / 2) for t in ts]
    # Chebyshev coefficients
    c = []
    for j in range(n):
        s = mp.fsum(ys[k] * mp.cos(j * mp.pi * (k + mp.mpf(1) / 2) / n) for k in range(n))
        c.append(s * (2 if j else 1) / n)
    # to monomials in t
    T = [[mp.mpf(1)], [mp.mpf(0), mp.mpf(1)]]
    for j in range(2, n):
        prev, pp = T[-1], T[-2]
        nxt = [mp.mpf(0)] * (j + 1)
        for i, v in enumerate(prev):
            nxt[i + 1] += 2 * v
        for i, v in enumerate(pp):
            nxt[i] -= v
        T.append(nxt)
    mono = [mp.mpf(0)] * n
    for j in range(n):
        for i, v in enumerate(T[j]):
            mono[i] += c[j] * v
    return [float(v) for v in mono]


def horner(p, t):
    r = 0.0
    for v in reversed(p):
        r = r * t + v
    return r


tab = [fit(i * W) for i in range(NI)]
worst = 0.0
for i in range(NI):
    for x in np.linspace(i * W, (i + 1) * W, 400, endpoint=False):
        t = (x - i * W) * (2 / W) - 1.0
        got = horner(tab[i], t)
        worst = max(worst, abs(got / float(erfcx(x)) - 1))
print(f"// max relative error of the double-precision Horner: {worst:.2e}")
print("__constant__ double c_erfcx_tab[%d][%d] = {" % (NI, DEG + 1))
for p in tab:
    print("    {" + ", ".join(repr(v) for v in p) + "},")
print("};")
