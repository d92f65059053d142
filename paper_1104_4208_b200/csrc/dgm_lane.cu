// Lane-pair stage kernels for low orders (p <= kLanePmax), sm_100a FP64.
//
// A warp owns 16 consecutive elements; lanes e and e+16 form the pair that
// works on element e0+e (half h = lane>>4).  The elements' coefficient blocks
// are contiguous in the SoA arrays, so they move with fully coalesced accesses
// into shared memory with an element-major layout s[e*SE + slot], SE odd (the 16
// lanes of a half-warp then hit 16 distinct bank pairs).  Both halves run the same generated code (gen/lanegen.py) on
// different components, so there is no divergence:
//   curl     ∂x: (Ŷz → -ĉy | Ŷy → +ĉz)  ∂y: (Ŷz → +ĉx | Ŷx → -ĉz)  ∂z: (Ŷy → -ĉx | Ŷx → +ĉy)
//   traces   half h: a_h = Ŷ·t̂_h on each face
//   lift     half 0: B = sf D₁ (+ upwind), half 1: A = -sf D₂ (+ upwind);
//            acc_m += t̂1_m L_f(A) + t̂2_m L_f(B)
// Own and neighbour traces come from a trace buffer written by the stage that
// updated that field (no neighbour volume reads).  Its layout interleaves groups
// of 16 elements, tr[e/16][f][k][γ][e%16], so the own-trace loads and the
// trace stores of a half-warp are single 128-byte transactions.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "dgm_internal.h"
#include "lane/lane_p1.cuh"
#include "lane/lane_p2.cuh"
#include "lane/lane_p3.cuh"
#include "lane/lane_p4.cuh"
#include "lane/lane_p5.cuh"
#include "lane/lane_p6.cuh"

namespace dgm {

__host__ __device__ constexpr int odd_up(int x) { return x | 1; }

template <int P>
struct L2 {
  static constexpr int N = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NF = (P + 1) * (P + 2) / 2;
  static constexpr int LD = (N + 3) & ~3;
  // per element: Ŷ (then X) with component stride LD (the padding modes are staged
  // too, so full groups copy without predicates), then the accumulator (stride N)
  static constexpr int SY = 0, SA = 3 * LD;
  static constexpr int SE = odd_up(3 * LD + 3 * N);  // per-element stride (odd: conflict-free)
  static constexpr int WS = 16 * SE;               // doubles per warp
  static constexpr int J = (16 * LD + 31) / 32;    // 8-byte copies per lane per component
  static constexpr int WARPS_RAW = (200 * 1024) / (WS * 8);
  static constexpr int WARPS = WARPS_RAW < 1 ? 1 : (WARPS_RAW > 8 ? 8 : WARPS_RAW);
};

#define DGM_L2_OPS(P)                                                                                     \
  template <>                                                                                             \
  struct LOps<P> {                                                                                        \
    static __device__ __forceinline__ void sweep(int d, const double *src, double *dst, double sgn) {     \
      if (d == 0) lane_sweep_p##P##_d0(src, dst, sgn);                                                    \
      else if (d == 1) lane_sweep_p##P##_d1(src, dst, sgn);                                               \
      else lane_sweep_p##P##_d2(src, dst, sgn);                                                           \
    }                                                                                                     \
    static __device__ __forceinline__ void trace(int f, const double *a, const double *b, double *out,    \
                                                 int os) {                                                \
      if (f == 0) lane_trace_p##P##_f0(a, b, out, os);                                                    \
      else if (f == 1) lane_trace_p##P##_f1(a, out, os);                                                  \
      else if (f == 2) lane_trace_p##P##_f2(a, out, os);                                                  \
      else lane_trace_p##P##_f3(a, out, os);                                                              \
    }                                                                                                     \
    template <int NF>                                                                                     \
    static __device__ __forceinline__ void lift(int f, const double (&q)[NF], double *o, double *o0,      \
                                                int h) {                                                  \
      lane_lift_p##P(f, q, o, o0, h);                                                                     \
    }                                                                                                     \
  };

template <int P>
struct LOps;
DGM_L2_OPS(1)
DGM_L2_OPS(2)
DGM_L2_OPS(3)
DGM_L2_OPS(4)
DGM_L2_OPS(5)
DGM_L2_OPS(6)

// tangential component h of face f: a_h = Y[c] (- Y[0] on face 0)
__device__ __forceinline__ int tang_comp(int f, int h) {
  return f == 0 ? 1 + h : (f == 1 ? 1 + h : (f == 2 ? 2 * h : h));
}
// lift destination component of half h on faces 1..3 (t̂ entries are +1 there)
__device__ __forceinline__ int lift_dst(int f, int h) {
  return f == 1 ? (h ? 1 : 2) : (f == 2 ? (h ? 0 : 2) : (h ? 0 : 1));
}

__device__ __forceinline__ void cp_async8(double *smem_dst, const double *gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Per-lane destination offsets of the flat copy of 16 element blocks (16*LD
// contiguous doubles per component): flat index i = lane + 32 j -> element i/LD,
// mode i%LD; -1 marks padding modes.  Computed once per kernel.
template <int N, int LD, int SE, int J>
struct CopyMap {
  int off[J];
  unsigned long long real;   // bit j: copy j carries a real mode (b < N); stores skip padding
  static_assert(J <= 64, "copy mask is 64 bits");
  __device__ __forceinline__ CopyMap(int lane) {
    real = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int i = lane + 32 * j, e = i / LD, b = i - e * LD;
      off[j] = e * SE + b;
      if (b < N && e < 16) real |= 1ull << j;
    }
  }
};

// Coalesced asynchronous load (cp.async, LDGSTS) of nel contiguous element blocks
// per component into s[e*SE + c*LD + b] (padding modes included); every copy of the
// group is in flight at once; the caller waits with cp_async_wait_all + __syncwarp.
template <int N, int LD, int SE, int J>
__device__ __forceinline__ void l2_load_async(const CopyMap<N, LD, SE, J> &m, const double *__restrict__ F,
                                              int64_t e0, int nel, int64_t cs, double *s, int lane) {
  if (nel == 16) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double *src = F + c * cs + e0 * LD + lane;
#pragma unroll
      for (int j = 0; j < J; ++j)
        if (32 * j + 31 < 16 * LD || lane + 32 * j < 16 * LD) cp_async8(s + c * LD + m.off[j], src + 32 * j);
    }
  } else {
    const int lim = nel * LD - lane;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double *src = F + c * cs + e0 * LD + lane;
#pragma unroll
      for (int j = 0; j < J; ++j)
        if (32 * j < lim) cp_async8(s + c * LD + m.off[j], src + 32 * j);
    }
  }
}

template <int N, int LD, int SE, int J>
__device__ __forceinline__ void l2_load(const CopyMap<N, LD, SE, J> &m, const double *__restrict__ F, int64_t e0,
                                        int nel, int64_t cs, double *s, int lane) {
  l2_load_async(m, F, e0, nel, cs, s, lane);
  cp_async_wait_all();
}

// store of the real modes (padding untouched)
template <int N, int LD, int SE, int J>
__device__ __forceinline__ void l2_store(const CopyMap<N, LD, SE, J> &m, double *__restrict__ F, int64_t e0, int nel,
                                         int64_t cs, const double *s, int lane, bool accumulate) {
  const int nj = (nel * LD - lane + 31) / 32;   // copies of this lane inside the group (nel >= 1)
  const unsigned long long mask = nel == 16 || nj >= J ? m.real : m.real & ((1ull << nj) - 1ull);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double *dst = F + c * cs + e0 * LD + lane;
    const double *src = s + c * LD;
#pragma unroll
    for (int j = 0; j < J; ++j)
      if ((mask >> j) & 1ull) {
        const double v = src[m.off[j]];
        dst[32 * j] = accumulate ? dst[32 * j] + v : v;
      }
  }
}

// trace-buffer index of (element ge, face f, component k, mode γ): groups of 16
// elements interleaved, tr[ge/16][f][k][γ][ge%16]
template <int NF>
__device__ __forceinline__ int64_t tix(int64_t ge, int f, int k, int g) {
  return (((ge >> 4) * 8 * NF + (f * 2 + k) * NF + g) << 4) + (ge & 15);
}

// traces of this lane's element (slots [0,3N)): tangential component h of all 4
// faces, written straight to the (interleaved, coalesced) trace buffer
template <int P>
__device__ __forceinline__ void l2_traces_out(const double *el, int h, double *__restrict__ tr, int64_t ge) {
  using D = L2<P>;
#pragma unroll 1
  for (int f = 0; f < 4; ++f) {
    const int c = tang_comp(f, h);
    LOps<P>::trace(f, el + c * D::LD, el, tr + tix<D::NF>(ge, f, h, 0), 16);
  }
}

template <int P, bool UP>
__global__ void __launch_bounds__(L2<P>::WARPS * 32)
    lane_stage_kernel(StageArgs a, const double *__restrict__ trY, double *__restrict__ trOut) {
  using D = L2<P>;
  constexpr int N = D::N, NF = D::NF, LD = D::LD;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;   // chosen at launch (<= D::WARPS) to balance the last round
  const int e = lane & 15, h = lane >> 4;
  double *sw = smem + warp * D::WS;
  double *el = sw + e * D::SE;
  const CopyMap<N, LD, D::SE, D::J> cmap(lane);
  const int64_t cs = a.n_tet * LD;
  const bool stageE = a.stage == STAGE_E;
  const bool upd = a.out_mode == OUT_UPDATE;
  // curl split: (source comp, destination comp, sign) per direction and half
  const int csrc0 = h ? 1 : 2, cdst0 = h ? 2 : 1;   // ∂x: (Ŷz → -ĉy | Ŷy → +ĉz)
  const int csrc1 = h ? 0 : 2, cdst1 = h ? 2 : 0;   // ∂y: (Ŷz → +ĉx | Ŷx → -ĉz)
  const int csrc2 = h ? 0 : 1, cdst2 = h ? 1 : 0;   // ∂z: (Ŷy → -ĉx | Ŷx → +ĉy)
  const double cs0 = h ? 1.0 : -1.0, cs1 = h ? -1.0 : 1.0, cs2 = h ? 1.0 : -1.0;
  for (int64_t e0 = ((int64_t)blockIdx.x * nwarps + warp) * 16; e0 < a.n_tet;
       e0 += (int64_t)gridDim.x * nwarps * 16) {
    const int nel = (int)(a.n_tet - e0 < 16 ? a.n_tet - e0 : 16);
    const bool active = e < nel;
    const int64_t ge = e0 + e;
    l2_load(cmap, a.Y, e0, nel, cs, sw, lane);
    {
      double *z = el + D::SA + h;
#pragma unroll
      for (int i = 0; i < (3 * N + 1) / 2; ++i)
        if (2 * i + 1 < 3 * N || h == 0) z[2 * i] = 0.0;
    }
    __syncwarp();
    // own and neighbour traces of this half's component (written by the stage that
    // last updated Ŷ), prefetched one face ahead
    double ownv[NF], nbv[NF];
    auto fetch = [&](int f) {
      if (!active) return;
      const double *to = trY + tix<NF>(ge, f, h, 0);
#pragma unroll
      for (int gm = 0; gm < NF; ++gm) ownv[gm] = __ldg(to + 16 * gm);
      const int nb = a.nbr[4 * ge + f];
      if (nb >= 0) {
        const double *tn = trY + tix<NF>(nb, a.nbrf[4 * ge + f], h, 0);
#pragma unroll
        for (int gm = 0; gm < NF; ++gm) nbv[gm] = __ldg(tn + 16 * gm);
      }
    };
    if (a.do_flux) fetch(0);   // face-0 gathers overlap the curl
    if (a.do_curl) {
      LOps<P>::sweep(0, el + csrc0 * LD, el + D::SA + cdst0 * N, cs0);
      __syncwarp();
      LOps<P>::sweep(1, el + csrc1 * LD, el + D::SA + cdst1 * N, cs1);
      __syncwarp();
      LOps<P>::sweep(2, el + csrc2 * LD, el + D::SA + cdst2 * N, cs2);
      __syncwarp();
    }
    bool x_issued = false;
    if (a.do_flux) {
      Geo g;
      double sgn = 1.0;
      if (active) {
        g = a.geo[ge];
        sgn = g.detF > 0 ? 1.0 : -1.0;
      }
      const double mirrorY = stageE ? 1.0 : -1.0, mirrorX = stageE ? -1.0 : 1.0;
      if (upd) {
        // the curl is done with Ŷ (and the fluxes only need traces): fetch X into
        // its slots now so the copy overlaps the four face fluxes and lifts
        l2_load_async(cmap, a.X, e0, nel, cs, sw, lane);
        x_issued = true;
      }
#pragma unroll 1
      for (int f = 0; f < 4; ++f) {
        double q[NF], cur[NF];
#pragma unroll
        for (int gm = 0; gm < NF; ++gm) {
          q[gm] = ownv[gm];
          cur[gm] = nbv[gm];
        }
        if (f < 3) fetch(f + 1);
        if (active) {
          const int nb = a.nbr[4 * ge + f];
          const int gf = a.nbrf[4 * ge + f];
          double w = 0.5, k = 0.0;
          if (UP) {
            const double Zm = g.Z, Zp = nb >= 0 ? a.geo[nb].Z : Zm;
            if (stageE) {
              w = Zp / (Zm + Zp);
              k = 1.0 / (Zm + Zp);
            } else {
              const double Ym = 1.0 / Zm, Yp = 1.0 / Zp;
              w = Yp / (Ym + Yp);
              k = 1.0 / (Ym + Yp);
            }
          }
          const double sf = (f & 1) ? -1.0 : 1.0;
          const double fs = h ? -sf : sf;   // half 0: B = sf D1, half 1: A = -sf D2
          double M0 = 0, M1 = 0, M2 = 0, ps = 0;
          const double *xo = nullptr, *xn = nullptr;
          if (UP) {
            const double *M = a.fmet + 12 * ge + 3 * f;
            M0 = M[0], M1 = M[1], M2 = M[2];
            ps = (stageE ? 1.0 : -1.0) * sgn;
            xo = a.trX + tix<NF>(ge, f, 0, 0);
            xn = nb >= 0 ? a.trX + tix<NF>(nb, gf, 0, 0) : nullptr;
          }
          // stabilised flux (E stage): the face unknown enters as Δ_k -= H^F_k
          const double *hfp = a.HF ? a.HF + ((int64_t)a.fid[4 * ge + f] * 2 + h) * NF : nullptr;
#pragma unroll
          for (int gm = 0; gm < NF; ++gm) {
            const double t = q[gm];
            const double tnv = nb >= 0 ? cur[gm] : mirrorY * t;
            double v = fs * (w * (tnv - t) - (hfp ? __ldg(hfp + gm) : 0.0));
            if (UP) {
              const double xo1 = __ldg(xo + 16 * gm), xo2 = __ldg(xo + 16 * (NF + gm));
              const double xn1 = nb >= 0 ? __ldg(xn + 16 * gm) : mirrorX * xo1;
              const double xn2 = nb >= 0 ? __ldg(xn + 16 * (NF + gm)) : mirrorX * xo2;
              const double j1 = k * (xn1 - xo1), j2 = k * (xn2 - xo2);
              v += ps * (h ? (j1 * M0 + j2 * M1) : (j1 * M1 + j2 * M2));
            }
            q[gm] = v;
          }
        }
        // face 0: t̂1 = (-1,1,0), t̂2 = (-1,0,1): acc1 += A, acc2 += B, acc0 -= A+B;
        // faces 1-3: one destination component per half
        const int dst = f == 0 ? (h ? 1 : 2) : lift_dst(f, h);
        LOps<P>::lift(f, q, el + D::SA + dst * N, el + D::SA, h);
        __syncwarp();
      }
    }
    // S2 + S6: inverse mass with geometry, update or write; slots [0,3N) stage X / dX
    if (upd) {
      if (x_issued) {
        cp_async_wait_all();
      } else {
        __syncwarp();
        l2_load(cmap, a.X, e0, nel, cs, sw, lane);
      }
    }
    __syncwarp();
    if (active) {
      const Geo g = a.geo[ge];
      const double cm = stageE ? g.inv_eps : -g.inv_mu;
      const double sc = upd ? a.dt * cm : cm;
      const double *ac = el + D::SA + h;
      double *xs = el + h;
      constexpr int UNR = N <= 40 ? (N + 1) / 2 : 4;   // full unroll only while the code stays small
#pragma unroll UNR
      for (int bb = 0; bb < (N + 1) / 2; ++bb) {
        if (2 * bb + 1 < N || h == 0) {   // mode b = 2bb + h
          const double v0 = ac[2 * bb], v1 = ac[N + 2 * bb], v2 = ac[2 * N + 2 * bb];
          const double x0 = sc * (g.g[0] * v0 + g.g[1] * v1 + g.g[2] * v2);
          const double x1 = sc * (g.g[1] * v0 + g.g[3] * v1 + g.g[4] * v2);
          const double x2 = sc * (g.g[2] * v0 + g.g[4] * v1 + g.g[5] * v2);
          if (upd) {
            xs[2 * bb] += x0;
            xs[LD + 2 * bb] += x1;
            xs[2 * LD + 2 * bb] += x2;
          } else {
            xs[2 * bb] = x0;
            xs[LD + 2 * bb] = x1;
            xs[2 * LD + 2 * bb] = x2;
          }
        }
      }
    }
    __syncwarp();
    if (upd) {
      l2_store(cmap, a.X, e0, nel, cs, sw, lane, false);
      if (trOut && active) l2_traces_out<P>(el, h, trOut, ge);
    } else {
      l2_store(cmap, a.dX, e0, nel, cs, sw, lane, a.out_mode == OUT_ACCUM);
    }
    __syncwarp();
  }
}

template <int P>
__global__ void __launch_bounds__(L2<P>::WARPS * 32)
    lane_trace_kernel(const double *__restrict__ X, double *__restrict__ tr, int64_t n_tet) {
  using D = L2<P>;
  constexpr int N = D::N, NF = D::NF, LD = D::LD;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = lane & 15, h = lane >> 4;
  double *sw = smem + warp * D::WS;
  const CopyMap<N, LD, D::SE, D::J> cmap(lane);
  const int64_t cs = n_tet * LD;
  for (int64_t e0 = ((int64_t)blockIdx.x * D::WARPS + warp) * 16; e0 < n_tet; e0 += (int64_t)gridDim.x * D::WARPS * 16) {
    const int nel = (int)(n_tet - e0 < 16 ? n_tet - e0 : 16);
    l2_load(cmap, X, e0, nel, cs, sw, lane);
    __syncwarp();
    if (e < nel) l2_traces_out<P>(sw + e * D::SE, h, tr, e0 + e);
    __syncwarp();
  }
}

template <typename K>
static int occupancy_grid(dgm_ctx *c, K kernel, int warps, size_t smem, int64_t groups) {
  int occ = 0;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, warps * 32, smem);
  if (occ < 1) occ = 1;
  int64_t grid = (groups + warps - 1) / warps;
  if (grid > (int64_t)c->sms * occ) grid = (int64_t)c->sms * occ;
  return (int)grid;
}

// Warps per CTA for n_tet elements: the persistent grid gives every warp a fixed
// sequence of 16-element groups, so the last round can be nearly empty.  Pick w
// minimising rounds(w) * w^0.55 (per-SM throughput measured to grow ~ w^0.45).
static int pick_warps(int64_t n_tet, int sms, int wmax, int ctas_per_sm_for_w1) {
  if (const char *v = std::getenv("DGM_LANE_WARPS")) {   // experiments only
    const int w = std::atoi(v);
    if (w >= 1 && w <= wmax) return w;
  }
  const int64_t groups = (n_tet + 15) / 16;
  double best = 1e300;
  int bw = wmax;
  for (int w = 1; w <= wmax; ++w) {
    const int64_t slots = (int64_t)sms * w;
    const double rounds = (double)((groups + slots - 1) / slots);
    const double cost = rounds * std::pow((double)w, 0.55);
    if (cost < best - 1e-9) {
      best = cost;
      bw = w;
    }
  }
  (void)ctas_per_sm_for_w1;
  return bw;
}

template <int P>
static dgm_status lane_stage_p(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st) {
  using D = L2<P>;
  const int w = pick_warps(c->n_tet, c->sms, D::WARPS, 1);
  const size_t smem = sizeof(double) * D::WS * w;
  auto go = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * D::WS * D::WARPS));
    const int64_t groups = (c->n_tet + 15) / 16;
    int64_t grid = (groups + w - 1) / w;
    if (grid > c->sms) grid = c->sms;   // one CTA of w warps per SM (shared memory bound)
    kernel<<<(unsigned)grid, w * 32, smem, st>>>(a, trY, trOut);
  };
  if (a.upwind) go(lane_stage_kernel<P, true>);
  else go(lane_stage_kernel<P, false>);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, DGM_ECUDA, std::string("lane_stage_kernel: ") + cudaGetErrorString(e));
  return DGM_OK;
}

template <int P>
static dgm_status lane_trace_p(dgm_ctx *c, const double *X, double *tr, cudaStream_t st) {
  using D = L2<P>;
  const size_t smem = sizeof(double) * D::WS * D::WARPS;
  const int grid = occupancy_grid(c, lane_trace_kernel<P>, D::WARPS, smem, (c->n_tet + 15) / 16);
  lane_trace_kernel<P><<<grid, D::WARPS * 32, smem, st>>>(X, tr, c->n_tet);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, DGM_ECUDA, std::string("lane_trace_kernel: ") + cudaGetErrorString(e));
  return DGM_OK;
}

dgm_status launch_lane_stage(dgm_ctx *c, int stage, const double *Y, double *X, double *dX, double dt, int do_curl,
                             int do_flux, int out_mode, const double *trY, const double *trX, double *trOut,
                             cudaStream_t st) {
  if (c->n_tet == 0) return DGM_OK;
  StageArgs a;
  a.Y = Y;
  a.X = X;
  a.dX = dX;
  a.trX = trX;
  a.geo = c->d_geo;
  a.nbr = c->d_nbr;
  a.nbrf = c->d_nbrf;
  a.fmet = c->d_fmet;
  a.n_tet = c->n_tet;
  a.dt = dt;
  a.stage = stage;
  a.upwind = c->flux == DGM_FLUX_UPWIND && do_flux;
  a.HF = (stage == STAGE_E && do_flux) ? c->cur_HF : nullptr;
  a.fid = c->d_fid;
  a.do_curl = do_curl;
  a.do_flux = do_flux;
  a.out_mode = out_mode;
  switch (c->p) {
    case 1: return lane_stage_p<1>(c, a, trY, trOut, st);
    case 2: return lane_stage_p<2>(c, a, trY, trOut, st);
    case 3: return lane_stage_p<3>(c, a, trY, trOut, st);
    case 4: return lane_stage_p<4>(c, a, trY, trOut, st);
    case 5: return lane_stage_p<5>(c, a, trY, trOut, st);
    case 6: return lane_stage_p<6>(c, a, trY, trOut, st);
  }
  return DGM_EORDER;
}

dgm_status launch_lane_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st) {
  if (c->n_tet == 0) return DGM_OK;
  switch (c->p) {
    case 1: return lane_trace_p<1>(c, X, tr, st);
    case 2: return lane_trace_p<2>(c, X, tr, st);
    case 3: return lane_trace_p<3>(c, X, tr, st);
    case 4: return lane_trace_p<4>(c, X, tr, st);
    case 5: return lane_trace_p<5>(c, X, tr, st);
    case 6: return lane_trace_p<6>(c, X, tr, st);
  }
  return DGM_EORDER;
}

}  // namespace dgm
