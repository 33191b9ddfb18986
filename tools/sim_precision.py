"""Numerics simulation behind the IMMA decode's operand precisions (float64 numpy, no GPU).

Quantizes K/V to 1-bit codes (the reference's channel-wise min/max quantizer), then compares
the calibrated decode output computed (a) exactly from the codes and (b) with the query
folded to `qbits`-bit integers and the probabilities to `pbits`-bit integers normalised per
`grp`-token group (power-of-two group scale), as the kernel does. Prints the worst relative
L2 error over heads and repetitions for each setting.
    python tools/sim_precision.py
"""
import numpy as np

rng = np.random.default_rng(7)


def run(n=4096, d=128, tau=(1.0, 0.0), qbits=15, pbits=16, grp=256, dist="gauss", qscale=1.0):
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, d))
    if dist == "t":
        k, v = rng.standard_t(3, size=(n, d)), rng.standard_t(3, size=(n, d))
    if dist == "outlier":  # the reference workload generator's outlier_channels flavour
        k[:, :4] *= 20
        v[:, :4] *= 20
    ka, kb = k.min(0), k.max(0)
    va, vb = v.min(0), v.max(0)
    kc = np.round((k - ka) / (kb - ka))
    vc = np.round((v - va) / (vb - va))
    vd = va + vc * (vb - va)
    errs = []
    for _ in range(4):
        q = rng.normal(size=d) * qscale
        qs, qa = q * (kb - ka), q @ ka

        def cal(s):
            gam, dl = s.min(), s.max()
            r = (tau[1] - tau[0]) / (dl - gam)
            return (1 - r) * s + r * gam - tau[0]

        z = cal((kc @ qs + qa) / np.sqrt(d))
        p = np.exp(z - z.max())
        o_ref = (p @ vd) / p.sum()
        S = (2 ** qbits - 1) / np.abs(qs).max()
        z = cal((kc @ (np.round(qs * S) / S) + qa) / np.sqrt(d))
        P = np.zeros(n)
        for w0 in range(0, n, grp):
            zw = z[w0:w0 + grp]
            mw = np.ceil((zw.max() - z.max()) / np.log(2)) * np.log(2)
            P[w0:w0 + grp] = np.round(np.exp(zw - z.max() - mw) * (2 ** pbits - 1)) * np.exp(mw)
        o = (P @ vd) / P.sum()
        errs.append(np.linalg.norm(o - o_ref) / np.linalg.norm(o_ref))
    return max(errs)


if __name__ == "__main__":
    cases = [dict(qbits=30, pbits=16, grp=1 << 20), dict(qbits=30, pbits=16, grp=1024), dict(qbits=30, pbits=16, grp=128),
             dict(qbits=15, pbits=24), dict(qbits=23, pbits=24), dict(qbits=15, pbits=24, dist="outlier"),
             dict(qbits=23, pbits=24, dist="outlier"), dict(qbits=30, pbits=16, grp=128, dist="outlier"),
             dict(qbits=30, pbits=16, grp=128, n=32768), dict(qbits=30, pbits=16, grp=128, dist="t")]
    for kw in cases:
        print(kw, f"{max(run(**kw) for _ in range(2)):.2e}")
