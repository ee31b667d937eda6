"""Certify-or-fallback feasibility with the bounds a kernel can afford (crude dropped-pair and residual
bounds from patch sums, the chain bound from one extra top-digit GEMM): fraction of ip1 outputs certified
and of (8-channel group, pixel) columns left for the exact DMMA recompute. Needs oracle/_ref (dev container)."""
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
# reuse the feasibility script's data preparation
src = open('tools/ozaki_feasibility.py').read()
src = src[:src.index('er=np.ceil')]
exec(src)
K = 19200
er = np.ceil(np.log2(np.abs(Wm).max(1))) + 1          # max|W_r| < 2^(er-1)
F = np.ceil(np.log2(col.max() * 256 / 255)) + 0      # max X < 2^F * 255/256 -> e0 <= 254
def wdig(S):
    N = np.rint(Wm * 2.0 ** (8 * S - er[:, None])).astype(np.int64)
    D = []; R = N.copy()
    for s in range(S - 1, 0, -1):
        D.append(R & 255); R = R >> 8
    D.append(R); return D[::-1]
def xdig(T):
    M = np.floor(col * 2.0 ** (8 * T - F)).astype(np.int64)
    E = []; R = M.copy()
    for t in range(T):
        E.append(R & 255); R = R >> 8
    return E[::-1]
gam = K * 2.0 ** -53 / (1 - K * 2.0 ** -53)
b32 = b.astype(np.float32)
yref = np.maximum((acc.astype(np.float32) + b32[:, None]).astype(np.float32), 0)
W1 = np.abs(Wm).sum(1); Xs = col.sum(0)
for S, T, L in [(6, 6, 5), (6, 6, 6), (7, 7, 6), (7, 7, 7)]:
    D = wdig(S); E = xdig(T)
    Esum = [e.sum(0).astype(np.float64) for e in E]     # per pixel patch sums of digit planes
    approx = np.zeros_like(acc); drop = np.zeros_like(acc); npairs = 0
    for s in range(S):
        for t in range(T):
            sc = 2.0 ** (er[:, None] + F - 8 * (s + t + 2))
            if s + t <= L:
                approx += (D[s].astype(np.float64) @ E[t].astype(np.float64)) * sc; npairs += 1
            else:
                drop += sc * (128.0 if s == 0 else 255.0) * Esum[t][None, :]
    # |w||x| upper bound from the top digits: (|d0|+1)(e0+1) * 2^(er+F-16)
    absb = ((np.abs(D[0]) + 1).astype(np.float64) @ (E[0] + 1).astype(np.float64)) * 2.0 ** (er[:, None] + F - 16)
    assert np.all(absb >= absum * (1 - 1e-12))
    bnd = drop + 2.0 ** (F - 8 * T) * W1[:, None] + 2.0 ** (er[:, None] - 8 * S - 1) * Xs[None, :]
    bnd += gam * absb + np.abs(approx) * 2.0 ** -50
    lo = (approx - bnd).astype(np.float32); hi = (approx + bnd).astype(np.float32)
    ylo = np.maximum((lo + b32[:, None]).astype(np.float32), 0); yhi = np.maximum((hi + b32[:, None]).astype(np.float32), 0)
    cert = ylo == yhi
    assert np.all(ylo[cert] == yref[cert])
    fails = ~cert
    g8 = fails.reshape(128, 8, -1).any(axis=1)   # (channel group of 8, pixel) columns needing exact recompute
    print(f"S{S} T{T} L{L}: {npairs}+1 int8 GEMMs, certified {cert.mean():.4f}, "
          f"fail {fails.mean():.4%} of outputs, (8-ch group, pixel) columns to recompute {g8.mean():.2%}")
