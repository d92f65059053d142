"""Where the dense engine's DMMA work goes: 16x8 block-granular FMA counts per
operator part (curl per direction, lift and trace per face) vs exact nonzeros.

usage: python tools/block_census.py [p ...]
Uses only the product-side generators (gen/plan.py programs on unit inputs).
"""
import sys
import numpy as np
from paper_1104_4208_b200.gen import plan

BK, BN = 16, 8
T1 = [(-1, 1, 0), (0, 1, 0), (1, 0, 0), (1, 0, 0)]
T2 = [(-1, 0, 1), (0, 0, 1), (0, 0, 1), (0, 1, 0)]


def blocks(M):
    """16-row x 8-column block-granular FMA count of M [K][Ncols] (rows padded)."""
    K, Nc = M.shape
    Kp, Np = -(-K // BK) * BK, -(-Nc // BN) * BN
    Z = np.zeros((Kp, Np), bool)
    Z[:K, :Nc] = M != 0
    b = Z.reshape(Kp // BK, BK, Np // BN, BN).any(axis=(1, 3))
    return int(b.sum()) * BK * BN, int(Z.sum())


def main():
    for p in [int(a) for a in sys.argv[1:]] or [6, 8, 10]:
        N, NF = plan.n_modes(p), plan.n_face_modes(p)
        # curl derivative matrices: D_d [N x N] (rows in, cols out) from unit inputs
        I = np.eye(N)
        res = {}
        tot_b = tot_e = 0
        for c in range(3):
            Y = np.zeros((3, N, N)); Y[c] = I
            C = plan.apply_curl_ref(p, Y)    # [3, n=N(unit idx), N]
            for m in range(3):
                M = C[m]                     # rows: unit input mode of comp c, cols: output mode
                M = np.where(np.abs(M) > 1e-13 * max(np.abs(M).max(), 1e-300), M, 0)
                if np.any(M):
                    b, e = blocks(M)
                    res[f"curl {c}->{m}"] = (b, e); tot_b += b; tot_e += e
        print(f"p={p} N={N} NF={NF}")
        print(f"  curl total: block {tot_b}  exact {tot_e}  (recurrence FMA {plan.fma_count_curl(p) if hasattr(plan,'fma_count_curl') else '?'})")
        for f in range(4):
            Tr = plan.apply_trace_ref(p, f, np.eye(N))   # [N, NF]
            Lf = plan.apply_lift_ref(p, f, np.eye(NF))   # [NF, N]
            # trace of tangential comps: rows 3N (component-blocked), cols 2 NF
            B2 = np.zeros((3 * N, 2 * NF))
            for k, t in enumerate((T1[f], T2[f])):
                for m in range(3):
                    if t[m]:
                        B2[m * N:(m + 1) * N, k * NF:(k + 1) * NF] = t[m] * Tr
            b2, e2 = blocks(B2)
            # lift: rows 2 NF (A, B), cols 3N: q_m = t1_m A + t2_m B
            B1 = np.zeros((2 * NF, 3 * N))
            for k, t in enumerate((T2[f], T1[f])):
                for m in range(3):
                    if t[m]:
                        B1[k * NF:(k + 1) * NF, m * N:(m + 1) * N] = Lf
            b1, e1 = blocks(B1)
            print(f"  face {f}: trace block {b2:7d} exact {e2:6d} | lift block {b1:7d} exact {e1:6d}")


main()
