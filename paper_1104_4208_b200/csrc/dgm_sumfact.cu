// Sum-factorised reverse numerical integration ("The 'reverse
// numerical integration' and the numerical integration used here can be accelerated by
// the use of the sum factorization technique ... O(p⁴)"), sm_100a FP64.
//
// The inverse mass of the point pipeline (variable materials, curved elements; readings
// G18, G19): residual coefficients acc (after the diagonal reference mass) -> values at
// the collapsed Gauss–Jacobi points -> per-point factor -> back to the modes.  With the
// collapsed coordinates (a, b, c) of the rule (x = (1+a)/2, y = (1-a)(1+b)/4,
// z = (1-a)(1-b)(1+c)/8) the basis of PAPER.md:785-789 factorises as
//     φ_ijk = P_i(c) · [((1-b)/2)^i P_j^{(2i+1,0)}(b)] · [((1-a)/2)^{i+j} P_k^{(2i+2j+2,0)}(a)]
//           = Pc[i](c) · Bb[i][j](b) · Ca[i+j][k](a),
// so the point values f(a_α, b_β, c_γ) = Σ_ijk acc_ijk φ_ijk are three one-dimensional
// contractions (k -> α, j -> β, i -> γ), each O(p⁴) per element instead of the O(p⁶)
// of the dense Φ (N x (p+2)³) the GEMM path applies, and the back transform is their
// transpose in reverse order.
//
// One CTA per group of EB = 256 / (p+2)² elements (grid-stride; EB = 1 from p = 9).  Per component the forward stages A, B write
// W[i][j][α] and U_c[i][α][β] to shared memory (inner dimension padded to an odd stride);
// one thread per point column (α, β) then runs stage C, the per-point factor (curved:
// symmetric 3x3 K_i; flat variable materials: the scalar ŵ_i / m(x_i)) and Cᵀ with the
// column's 3 x (p+2) point values in registers, overwriting U in place; Bᵀ (a thread per
// row (i, α), the row in registers) and Aᵀ leave the modal result in shared memory; the
// epilogue applies G' (flat) or nothing (curved, K carried it), the sign of the
// equation and the update X += dt Ẋ (or writes / accumulates dX).
// The 1D tables (host-built, dgm_host.cpp: sumfact_tables) are read through L1.
#include <cstdint>
#include <cstdlib>
#include <string>

#include "dgm_internal.h"

namespace dgm {
namespace {

template <int P>
struct SF {
  static constexpr int Q1 = P + 2;                  // points per direction
  static constexpr int QS = Q1 | 1;                 // padded (odd) inner stride
  static constexpr int N = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NP = (P + 1) * (P + 2) / 2;  // (i, j) pairs with i + j <= P
  static constexpr int W_SZ = (P + 1) * (P + 1) * QS;
  static constexpr int U_SZ = (P + 1) * Q1 * QS;
  static constexpr int EL = 3 * N + W_SZ + 3 * U_SZ;               // doubles per element
  static constexpr int EB = 256 / (Q1 * Q1) > 0 ? 256 / (Q1 * Q1) : 1;   // elements per CTA
  static constexpr int SMEM = 8 * EB * EL;
  // measured on a 10,368-tet curved cube (profiles/r02_sumfact_minb.txt): 3 CTAs per SM
  // (80 registers) is faster for p <= 5 and p = 10, 2 (128 registers) for p = 6..9
  static constexpr int MINB_DEFAULT = (P >= 6 && P <= 9) ? 2 : 3;
};

__device__ __forceinline__ int mode_index(int i, int j, int k) {
  const int n = i + j + k;
  return n * (n + 1) * (n + 2) / 6 + i * (n + 1) - i * (i - 1) / 2 + j;
}

template <int P, int MINB>
__global__ void __launch_bounds__(256, MINB) sumfact_kernel(SumfactArgs a) {
  using S = SF<P>;
  constexpr int Q1 = S::Q1, QS = S::QS, N = S::N, NP = S::NP, P1 = P + 1, EB = S::EB, EL = S::EL;
  extern __shared__ __align__(16) double sm[];
  // element slot l: acc [3][N] (residual, later the modal result), W [i][j][α] (one
  // component at a time), U [c][i][α][β]
  auto ACC = [&](int l) { return sm + l * EL; };
  auto WW = [&](int l) { return sm + l * EL + 3 * N; };
  auto UU = [&](int l) { return sm + l * EL + 3 * N + S::W_SZ; };
  const double *__restrict__ Pc = a.Pc;   // [i][γ]
  const double *__restrict__ Bb = a.Bb;   // [i][j][β]
  const double *__restrict__ Ca = a.Ca;   // [t][k][α]
  const int tid = threadIdx.x, T = blockDim.x;
  const int64_t cs = a.n_tet * (int64_t)a.LD;
  for (int64_t e0 = (int64_t)blockIdx.x * EB; e0 < a.n_tet; e0 += (int64_t)gridDim.x * EB) {
    const int nel = (int)(a.n_tet - e0 < EB ? a.n_tet - e0 : EB);
    for (int q = tid; q < nel * 3 * N; q += T) {
      const int l = q / (3 * N), r = q - l * 3 * N, c = r / N, b = r - c * N;
      ACC(l)[r] = a.AC[(e0 + l) * (int64_t)a.acld + c * a.acNk + b];
    }
    __syncthreads();
    // ---- forward A, B per component: modes -> U_c[i][α][β]
    for (int c = 0; c < 3; ++c) {
      // A (k -> α): W[i][j][α] = Σ_k Ca[i+j][k][α] v_ijk
      for (int o = tid; o < nel * NP * Q1; o += T) {
        const int l = o / (NP * Q1), r = o - l * NP * Q1, pr = r / Q1, al = r - pr * Q1;
        const double *v = ACC(l) + c * N;
        const int2 ij = a.pairs[pr];
        const int t = ij.x + ij.y, m0 = mode_index(ij.x, ij.y, 0);
        double s[2] = {0.0, 0.0};   // two partial sums: half the dependent-FMA chain
        const int t3 = t * (t + 1) * (t + 2);
        for (int k = 0; k <= P - t; ++k) {
          // mode (i, j, k) sits in degree block t + k, i (n - t) further on than (i, j, 0)
          const int n = t + k;
          s[k & 1] = fma(__ldg(Ca + (t * P1 + k) * Q1 + al), v[m0 + (n * (n + 1) * (n + 2) - t3) / 6 + ij.x * k], s[k & 1]);
        }
        WW(l)[(ij.x * P1 + ij.y) * QS + al] = s[0] + s[1];
      }
      __syncthreads();
      // B (j -> β): thread (i, α) computes the row U_c[i][α][0..q)
      for (int o = tid; o < nel * P1 * Q1; o += T) {
        const int l = o / (P1 * Q1), r = o - l * P1 * Q1, i = r / Q1, al = r - i * Q1;
        const double *W = WW(l);
        double *Uc = UU(l) + c * S::U_SZ;
        double rr[Q1];
#pragma unroll
        for (int be = 0; be < Q1; ++be) rr[be] = 0.0;
        for (int j = 0; j <= P - i; ++j) {
          const double w = W[(i * P1 + j) * QS + al];
          const double *bb = Bb + (i * P1 + j) * Q1;
#pragma unroll
          for (int be = 0; be < Q1; ++be) rr[be] = fma(__ldg(bb + be), w, rr[be]);
        }
#pragma unroll
        for (int be = 0; be < Q1; ++be) Uc[(i * Q1 + al) * QS + be] = rr[be];
      }
      __syncthreads();
    }
    // ---- C, the point factor and Cᵀ fused per column (α, β): the two lanes of a pair
    // take the column's first and second half of γ, hold those point values of the three
    // components in registers (point index (α q + β) q + γ, the host rule's order), and
    // combine their Cᵀ partial sums with one shuffle; U'_c[i][α][β] is written in place
    {
      constexpr int G2 = (Q1 + 1) / 2;
      const int count = nel * Q1 * Q1 * 2;
      for (int ob = 0; ob < count; ob += T) {   // uniform trip count: the shuffles need every lane
        const int o = ob + tid;
        const bool act = o < count;
        const int oc = act ? o >> 1 : 0, h = o & 1;
        const int l = oc / (Q1 * Q1), col = oc - l * Q1 * Q1, al = col / Q1, be = col - al * Q1;
        double *U = UU(l);
        const int g0 = h * G2;
        double f[3][G2];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int g = 0; g < G2; ++g) f[c][g] = 0.0;
        for (int i = 0; i <= P; ++i) {
          const int ui = (i * Q1 + al) * QS + be;
          const double u0 = U[ui], u1 = U[S::U_SZ + ui], u2 = U[2 * S::U_SZ + ui];
#pragma unroll
          for (int g = 0; g < G2; ++g)
            if (g0 + g < Q1) {
              const double pc = __ldg(Pc + i * Q1 + g0 + g);
              f[0][g] = fma(pc, u0, f[0][g]);
              f[1][g] = fma(pc, u1, f[1][g]);
              f[2][g] = fma(pc, u2, f[2][g]);
            }
        }
        const int64_t pt0 = (e0 + l) * (int64_t)a.Qk + (int64_t)col * Q1 + g0;
#pragma unroll
        for (int g = 0; g < G2; ++g) {
          if (!act || g0 + g >= Q1) continue;
          if (a.K) {
            const double *k = a.K + (pt0 + g) * 6;
            const double v0 = f[0][g], v1 = f[1][g], v2 = f[2][g];
            f[0][g] = k[0] * v0 + k[1] * v1 + k[2] * v2;
            f[1][g] = k[1] * v0 + k[3] * v1 + k[4] * v2;
            f[2][g] = k[2] * v0 + k[4] * v1 + k[5] * v2;
          } else {
            const double w = a.SW[pt0 + g];
            f[0][g] *= w;
            f[1][g] *= w;
            f[2][g] *= w;
          }
        }
        for (int i = 0; i <= P; ++i) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int g = 0; g < G2; ++g)
            if (g0 + g < Q1) {
              const double pc = __ldg(Pc + i * Q1 + g0 + g);
              s0 = fma(pc, f[0][g], s0);
              s1 = fma(pc, f[1][g], s1);
              s2 = fma(pc, f[2][g], s2);
            }
          s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
          s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
          if (act && h == (i & 1)) {   // the pair splits the stores
            const int ui = (i * Q1 + al) * QS + be;
            U[ui] = s0;
            U[S::U_SZ + ui] = s1;
            U[2 * S::U_SZ + ui] = s2;
          }
        }
      }
    }
    __syncthreads();
    // ---- back Bᵀ, Aᵀ per component
    for (int c = 0; c < 3; ++c) {
      // Bᵀ: thread (i, α) loads the row U'_c[i][α][0..q) and writes W[i][j][α] for all j
      for (int o = tid; o < nel * P1 * Q1; o += T) {
        const int l = o / (P1 * Q1), r = o - l * P1 * Q1, i = r / Q1, al = r - i * Q1;
        const double *Uc = UU(l) + c * S::U_SZ;
        double *W = WW(l);
        double rr[Q1];
#pragma unroll
        for (int be = 0; be < Q1; ++be) rr[be] = Uc[(i * Q1 + al) * QS + be];
        for (int j = 0; j <= P - i; ++j) {
          const double *bb = Bb + (i * P1 + j) * Q1;
          double s[3] = {0.0, 0.0, 0.0};
#pragma unroll
          for (int be = 0; be < Q1; ++be) s[be % 3] = fma(__ldg(bb + be), rr[be], s[be % 3]);
          W[(i * P1 + j) * QS + al] = s[0] + s[1] + s[2];
        }
      }
      __syncthreads();
      // Aᵀ: out_ijk = (1/‖φ_ijk‖²) Σ_α Ca[i+j][k][α] W[i][j][α]   (into acc_c)
      for (int o = tid; o < nel * N; o += T) {
        const int l = o / N, b = o - l * N;
        const int3 ijk = a.modes[b];
        const int t = ijk.x + ijk.y;
        const double *ca = Ca + (t * P1 + ijk.z) * Q1;
        const double *w = WW(l) + (ijk.x * P1 + ijk.y) * QS;
        double s[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int al = 0; al < Q1; ++al) s[al % 3] = fma(__ldg(ca + al), w[al], s[al % 3]);
        ACC(l)[c * N + b] = (s[0] + s[1] + s[2]) * __ldg(a.inv_norms + b);
      }
      __syncthreads();
    }
    // ---- epilogue: G' (flat) or none (curved, K carried it), the equation's sign, update/write
    const double cm = a.stageE ? 1.0 : -1.0;
    for (int o = tid; o < nel * N; o += T) {
      const int l = o / N, b = o - l * N;
      const int64_t e = e0 + l;
      const double *acc = ACC(l);
      const double v0 = acc[b], v1 = acc[N + b], v2 = acc[2 * N + b];
      double x0, x1, x2;
      if (a.K) {
        x0 = cm * v0;
        x1 = cm * v1;
        x2 = cm * v2;
      } else {
        const Geo &G = a.geo[e];
        x0 = cm * (G.g[0] * v0 + G.g[1] * v1 + G.g[2] * v2);
        x1 = cm * (G.g[1] * v0 + G.g[3] * v1 + G.g[4] * v2);
        x2 = cm * (G.g[2] * v0 + G.g[4] * v1 + G.g[5] * v2);
      }
      const int64_t off = e * (int64_t)a.LD + b;
      if (a.out_mode == OUT_UPDATE) {
        a.X[off] += a.dt * x0;
        a.X[cs + off] += a.dt * x1;
        a.X[2 * cs + off] += a.dt * x2;
      } else if (a.out_mode == OUT_ACCUM) {
        a.dX[off] += x0;
        a.dX[cs + off] += x1;
        a.dX[2 * cs + off] += x2;
      } else {
        a.dX[off] = x0;
        a.dX[cs + off] = x1;
        a.dX[2 * cs + off] = x2;
      }
    }
    __syncthreads();
  }
}

template <int P, int MINB>
dgm_status go_b(dgm_ctx *c, const SumfactArgs &a, cudaStream_t st) {
  constexpr int smem = SF<P>::SMEM;
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(sumfact_kernel<P, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sumfact_kernel<P, MINB>, 256, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t groups = (c->n_tet + SF<P>::EB - 1) / SF<P>::EB;
  int64_t grid = (int64_t)c->sms * occ;
  if (grid > groups) grid = groups;
  if (grid < 1) return DGM_OK;
  sumfact_kernel<P, MINB><<<(unsigned)grid, 256, smem, st>>>(a);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("sumfact_kernel: ") + cudaGetErrorString(e));
}

// CTAs per SM the register allocation targets (launch bounds): 3 (80 registers) or 2
// (128); DGM_SF_MINB=2|3 overrides for measurements
template <int P>
dgm_status go(dgm_ctx *c, const SumfactArgs &a, cudaStream_t st) {
  static int minb = 0;
  if (!minb) {
    minb = SF<P>::MINB_DEFAULT;
    if (const char *v = std::getenv("DGM_SF_MINB"))
      if (std::atoi(v) == 2 || std::atoi(v) == 3) minb = std::atoi(v);
  }
  return minb == 2 ? go_b<P, 2>(c, a, st) : go_b<P, 3>(c, a, st);
}

}  // namespace

dgm_status launch_sumfact(dgm_ctx *c, const SumfactArgs &a, cudaStream_t st) {
  switch (c->p) {
    case 1: return go<1>(c, a, st);
    case 2: return go<2>(c, a, st);
    case 3: return go<3>(c, a, st);
    case 4: return go<4>(c, a, st);
    case 5: return go<5>(c, a, st);
    case 6: return go<6>(c, a, st);
    case 7: return go<7>(c, a, st);
    case 8: return go<8>(c, a, st);
    case 9: return go<9>(c, a, st);
    case 10: return go<10>(c, a, st);
  }
  return set_err(c, DGM_EORDER, "sumfact: orders 1..10");
}

}  // namespace dgm
