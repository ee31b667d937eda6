"""CPU prototype of the exact-by-certification ip1 conv (DESIGN.md "Exact mode on integer tensor
cores"): the exact integer dot product of fixed-point weights and activations is computed as
int8 residue GEMMs modulo n pairwise-coprime moduli <= 256 and reconstructed by CRT; a rigorous
interval around it (fixed-point truncation + the reference chain's own rounding bound
gamma_K * sum|w x|) certifies float(acc) of the reference chain whenever both ends round to the
same float; everything else is recomputed by the exact chain.

Data: /tmp/feas.npz, /tmp/feas2.npz written by tools/ozaki_feasibility.py (the reference's own
pool3 / ip1 of sk.net on a 109x109 input, 65,536 ip1 outputs). Dev-container only.
"""
import math
import sys

import numpy as np

f1 = np.load("/tmp/feas.npz")
f2 = np.load("/tmp/feas2.npz")
Wm, col, acc = f2["Wm"], f2["col"], f2["acc"]  # [1024,19200] f64(f32 values), [19200,64], ref chain
b = f1["b10"].astype(np.float32)
M_, K = Wm.shape
yref = np.maximum((acc.astype(np.float32) + b[:, None]).astype(np.float32), 0)


def moduli(n):
    out = []
    p = 256
    while len(out) < n:
        if all(math.gcd(p, q) == 1 for q in out):
            out.append(p)
        p -= 1
    return out


def run(n, bw, bx, verbose=True):
    P_ = moduli(n)
    Mprod = math.prod(P_)
    # fixed point: Wi = rint(w * 2^sw_r), |Wi| <= 2^bw ; Xi = rint(x * 2^sx), 0 <= Xi <= 2^bx
    ew = np.ceil(np.log2(np.abs(Wm).max(1)))  # max|W_r| <= 2^ew
    sw = bw - ew
    ex = math.ceil(math.log2(col.max()))
    sx = bx - ex
    Wi = np.rint(Wm * 2.0 ** sw[:, None])   # exact in f64 (< 2^53)
    Xi = np.rint(col * 2.0 ** sx)
    assert np.abs(Wi).max() <= 2.0 ** bw and Xi.max() <= 2.0 ** bx
    assert K * 2.0 ** (bw + bx) < Mprod / 2, "moduli product too small"
    Wi64, Xi64 = Wi.astype(np.int64), Xi.astype(np.int64)
    # residue GEMMs (symmetric residues fit s8; |sum| <= K*128*128 < 2^31)
    res = []
    for p in P_:
        rw = ((Wi64 + p // 2) % p) - p // 2
        rx = ((Xi64 + p // 2) % p) - p // 2
        assert rw.min() >= -128 and rw.max() <= 127 and rx.min() >= -128 and rx.max() <= 127
        c = rw @ rx
        assert np.abs(c).max() < 2 ** 31
        res.append(c % p)
    # CRT: P = sum r_i c_i mod Mprod, c_i = (Mprod/p_i) * inv(Mprod/p_i mod p_i)
    cs = [(Mprod // p) * pow(Mprod // p, -1, p) for p in P_]
    Pint = np.zeros(res[0].shape, dtype=object)
    for r, c in zip(res, cs):
        Pint = Pint + r.astype(object) * c
    Pint = Pint % Mprod
    Pint = np.where(Pint > Mprod // 2, Pint - Mprod, Pint)
    # spot-check exactness against Python-int dot products
    for (i, j) in [(0, 0), (5, 17), (1023, 63), (400, 31)]:
        ex_ = sum(int(a) * int(c) for a, c in zip(Wi64[i], Xi64[:, j]))
        assert Pint[i, j] == ex_
    V = np.array([[float(v) for v in row] for row in Pint]) * 2.0 ** (-(sw[:, None] + sx))
    # bounds: truncation + chain rounding (sum|w x| from one u8 x u8 GEMM on 8-bit ceilings)
    W1 = (np.abs(Wi) * 2.0 ** -sw[:, None]).sum(1)           # sum |W~| per row
    X1 = Xi.sum(0) * 2.0 ** -sx + K * 2.0 ** (-sx - 1)         # >= sum |x| per pixel
    Et = 2.0 ** (-sw[:, None] - 1) * X1[None, :] + 2.0 ** (-sx - 1) * W1[:, None]
    Wa = np.ceil(np.abs(Wm) * 2.0 ** (8 - ew[:, None]))        # <= 256
    Wa = np.minimum(Wa, 255)  # |w| <= 2^ew * 255/256 needed: check
    assert np.all(np.abs(Wm) <= Wa * 2.0 ** (ew[:, None] - 8))
    Xa = np.ceil(col * 2.0 ** (8 - ex))
    Xa = np.minimum(Xa, 255)
    assert np.all(col <= Xa * 2.0 ** (ex - 8))
    Sabs = (Wa @ Xa) * 2.0 ** (ew[:, None] + ex - 16)
    absum = np.abs(Wm) @ np.abs(col)
    assert np.all(Sabs >= absum)
    gam = K * 2.0 ** -53 / (1 - K * 2.0 ** -53)
    E = Et + gam * Sabs + np.abs(V) * 2.0 ** -52
    lo = (V - E).astype(np.float32)
    hi = (V + E).astype(np.float32)
    ylo = np.maximum((lo + b[:, None]).astype(np.float32), 0)
    yhi = np.maximum((hi + b[:, None]).astype(np.float32), 0)
    cert = ylo == yhi
    assert np.all(ylo[cert] == yref[cert]), "certified output differs from the reference"
    ex_exact = f2["hi"] + f2["lo"]
    if verbose:
        print(f"n={n} moduli (M~2^{math.log2(Mprod):.1f}) bw={bw} bx={bx}: certified {cert.mean():.4%}, "
              f"fail {(~cert).mean():.4%}, pixels with a failure {(~cert).any(0).mean():.2%}, "
              f"max |V-exact|/Et {np.max(np.abs(V - ex_exact) / Et):.3f}, Et/(gam*Sabs) median "
              f"{np.median(Et / (gam * Sabs)):.3g}")
    return cert


if __name__ == "__main__":
    print("moduli:", moduli(16))
    for n, bw, bx in [(12, 40, 39), (13, 43, 43), (14, 47, 47), (15, 51, 51)]:
        try:
            run(n, bw, bx)
        except AssertionError as e:
            print(n, bw, bx, "FAILED:", e)
            sys.exit(1)
