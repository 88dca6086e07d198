"""Calibrate the far-field tensor Gauss order q(g), g = gap / max(diam_i, diam_j).

For seeded random panel pairs (coplanar / parallel-offset / orthogonal, aspect up
to 4, size ratio up to 8) at prescribed g, measure the relative error of the
q^4-point tensor Gauss-Legendre rule against a composite truth (q=10 rule on a
3x3 split of each panel).  Prints, per q, the largest error seen per g bin.
"""
import numpy as np, sys

def gl(q):
    x, w = np.polynomial.legendre.leggauss(q)
    return x, w

def inplane(axis):
    return {0: (1, 2), 1: (0, 2), 2: (0, 1)}[axis]

def gauss_pairs(P, Q, q, sub=1):
    # P, Q: arrays (N, 6) of axis, level, a0, a1, b0, b1
    x, w = gl(q)
    N = P.shape[0]
    tot = np.zeros(N)
    for si in range(sub):
        for sj in range(sub):
            for sk in range(sub):
                for sl in range(sub):
                    def pts(R, s1, s2):
                        ax = R[:, 0].astype(int)
                        a0 = R[:, 2] + (R[:, 3] - R[:, 2]) * s1 / sub
                        a1 = R[:, 2] + (R[:, 3] - R[:, 2]) * (s1 + 1) / sub
                        b0 = R[:, 4] + (R[:, 5] - R[:, 4]) * s2 / sub
                        b1 = R[:, 4] + (R[:, 5] - R[:, 4]) * (s2 + 1) / sub
                        ca, ha = (a0 + a1) / 2, (a1 - a0) / 2
                        cb, hb = (b0 + b1) / 2, (b1 - b0) / 2
                        A = ca[:, None] + ha[:, None] * x[None, :]   # N,q
                        B = cb[:, None] + hb[:, None] * x[None, :]
                        WA = ha[:, None] * w[None, :]
                        WB = hb[:, None] * w[None, :]
                        C = np.zeros((N, 3, q, q))
                        for n in range(N):
                            i0, i1 = inplane(ax[n])
                            C[n, ax[n]] = R[n, 1]
                            C[n, i0] = A[n][:, None]
                            C[n, i1] = B[n][None, :]
                        W = WA[:, :, None] * WB[:, None, :]
                        return C.reshape(N, 3, q * q), W.reshape(N, q * q)
                    CP, WP = pts(P, si, sj)
                    CQ, WQ = pts(Q, sk, sl)
                    d = CP[:, :, :, None] - CQ[:, :, None, :]
                    r = np.sqrt((d * d).sum(1))
                    tot += np.einsum('na,nb,nab->n', WP, WQ, 1.0 / r)
    return tot / (4 * np.pi)

def rect_dist(P, Q):
    def ext(R, k):
        lo = np.zeros(len(R)); hi = np.zeros(len(R))
        for n in range(len(R)):
            ax = int(R[n, 0]); i0, i1 = inplane(ax)
            if k == ax: lo[n] = hi[n] = R[n, 1]
            elif k == i0: lo[n], hi[n] = R[n, 2], R[n, 3]
            else: lo[n], hi[n] = R[n, 4], R[n, 5]
        return lo, hi
    s = 0
    for k in range(3):
        la, ha = ext(P, k); lb, hb = ext(Q, k)
        g = np.maximum(np.maximum(lb - ha, la - hb), 0)
        s = s + g * g
    return np.sqrt(s)

def diam(R):
    return np.hypot(R[:, 3] - R[:, 2], R[:, 5] - R[:, 4])

def gen(rng, N, gtarget):
    P = np.zeros((N, 6)); Q = np.zeros((N, 6))
    for n in range(N):
        while True:
            ax = rng.integers(3)
            la = rng.uniform(0.25, 1) ; lb = la * rng.uniform(0.25, 4) if rng.random() < 0.5 else la
            P[n] = [ax, 0, -la / 2, la / 2, -lb / 2, lb / 2]
            s = np.exp(rng.uniform(np.log(1 / 8), np.log(8)))
            la2 = rng.uniform(0.25, 1) * s; lb2 = la2 * rng.uniform(0.25, 4)
            cls = rng.integers(3)
            ax2 = ax if cls < 2 else (ax + 1 + rng.integers(2)) % 3
            # random direction, then scale offset to hit gtarget
            d = rng.normal(size=3); d /= np.linalg.norm(d)
            if cls == 0: d[ax] = 0; d /= max(np.linalg.norm(d), 1e-12)
            cen = d
            Q[n] = [ax2, 0, 0, 0, 0, 0]
            def place(t):
                c = cen * t
                i0, i1 = inplane(ax2)
                lev = c[ax2] if cls != 0 else 0.0
                return [ax2, lev, c[i0] - la2 / 2, c[i0] + la2 / 2, c[i1] - lb2 / 2, c[i1] + lb2 / 2]
            lo, hi = 0.0, 100.0
            dm = max(np.hypot(la, lb), np.hypot(la2, lb2))
            for _ in range(60):
                mid = 0.5 * (lo + hi)
                Q[n] = place(mid)
                g = rect_dist(P[n:n+1], Q[n:n+1])[0] / dm
                if g < gtarget: lo = mid
                else: hi = mid
            Q[n] = place(hi)
            if abs(rect_dist(P[n:n+1], Q[n:n+1])[0] / dm - gtarget) < 1e-3 * gtarget:
                break
    return P, Q

rng = np.random.default_rng(7)
gs = [float(a) for a in sys.argv[1:]] or [0.5, 0.75, 1.0, 1.5, 2, 3, 4, 6, 8, 12, 16, 24, 32, 64]
N = 300
for g in gs:
    P, Q = gen(rng, N, g)
    truth = gauss_pairs(P, Q, 10, sub=3)
    row = []
    for q in range(1, 11):
        v = gauss_pairs(P, Q, q)
        row.append(np.max(np.abs(v - truth) / truth))
    print("g=%6.2f " % g + " ".join("q%d:%.1e" % (q + 1, e) for q, e in enumerate(row)), flush=True)
