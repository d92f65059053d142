// Lane-per-element stage kernels for low orders (p <= DGM_LANE_PMAX), sm_100a FP64.
//
// A warp owns 32 consecutive elements.  Their coefficient blocks are contiguous
// in the SoA field arrays, so they are loaded/stored with fully coalesced
// accesses and transposed through shared memory into an element-interleaved
// layout s[slot*33 + lane] (conflict-free for the compute).  Every thread then
// runs the same generated straight-line program (gen/lanegen.py) on its own
// element: curl by the recurrence sweeps, traces, numerical flux, lift, inverse
// mass, update — coefficients are compile-time constants (warp-uniform).
// Neighbour traces come from a trace buffer tr[e][f][k][γ] that the previous
// stage wrote for the field it updated (the stage that updates X also emits
// X's traces), so no neighbour volume data is read.
#include <cstdint>

#include "dgm_internal.h"
#include "lane/lane_p1.cuh"
#include "lane/lane_p2.cuh"
#include "lane/lane_p3.cuh"
#include "lane/lane_p4.cuh"

namespace dgm {

constexpr int kLS = 33;   // interleave stride (doubles)

template <int P>
struct LDim {
  static constexpr int N = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NF = (P + 1) * (P + 2) / 2;
  static constexpr int LD = (N + 3) & ~3;
  static constexpr int SY = 3 * N;                               // Y, then X (or dX) staging
  static constexpr int SA = 3 * N > 8 * NF ? 3 * N : 8 * NF;    // accumulator, then X-traces
  static constexpr int WS = (SY + SA) * kLS;                     // doubles per warp
  static constexpr int WARPS_RAW = (200 * 1024) / (WS * 8);
  static constexpr int WARPS = WARPS_RAW < 1 ? 1 : (WARPS_RAW > 4 ? 4 : WARPS_RAW);
};

#define DGM_LANE_OPS(P)                                                                                    \
  template <>                                                                                              \
  struct LaneOps<P> {                                                                                      \
    static constexpr int NF = LDim<P>::NF;                                                                 \
    static __device__ __forceinline__ void curl(const double *sY, double *sA) { lane_curl_p##P(sY, sA); }  \
    template <int F>                                                                                       \
    static __device__ __forceinline__ void trace(const double *sY, double (&t)[2][NF]) {                   \
      if (F == 0) lane_trace_p##P##_f0(sY, t);                                                             \
      else if (F == 1) lane_trace_p##P##_f1(sY, t);                                                        \
      else if (F == 2) lane_trace_p##P##_f2(sY, t);                                                        \
      else lane_trace_p##P##_f3(sY, t);                                                                    \
    }                                                                                                      \
    template <int F>                                                                                       \
    static __device__ __forceinline__ void lift(const double (&q)[3][NF], double *sA) {                    \
      if (F == 0) lane_lift_p##P##_f0(q, sA);                                                              \
      else if (F == 1) lane_lift_p##P##_f1(q, sA);                                                         \
      else if (F == 2) lane_lift_p##P##_f2(q, sA);                                                         \
      else lane_lift_p##P##_f3(q, sA);                                                                     \
    }                                                                                                      \
  };

template <int P>
struct LaneOps;
DGM_LANE_OPS(1)
DGM_LANE_OPS(2)
DGM_LANE_OPS(3)
DGM_LANE_OPS(4)

__device__ __constant__ double kLT1[4][3] = {{-1, 1, 0}, {0, 1, 0}, {1, 0, 0}, {1, 0, 0}};
__device__ __constant__ double kLT2[4][3] = {{-1, 0, 1}, {0, 0, 1}, {0, 0, 1}, {0, 1, 0}};

// coalesced load of `rows` contiguous blocks of LD doubles (component stride cs)
// into the interleaved layout s[(c*N + b)*33 + e]
template <int N, int LD>
__device__ __forceinline__ void lane_load(const double *__restrict__ F, int64_t e0, int nel, int64_t cs, double *s,
                                          int lane) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double *src = F + c * cs + e0 * LD;
    for (int i = lane; i < nel * LD; i += 32) {
      const int e = i / LD, b = i - e * LD;
      if (b < N) s[(c * N + b) * kLS + e] = __ldg(src + i);
    }
  }
}

template <int N, int LD>
__device__ __forceinline__ void lane_store(double *__restrict__ F, int64_t e0, int nel, int64_t cs, const double *s,
                                           int lane, bool accumulate) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double *dst = F + c * cs + e0 * LD;
    for (int i = lane; i < nel * LD; i += 32) {
      const int e = i / LD, b = i - e * LD;
      if (b < N) {
        const double v = s[(c * N + b) * kLS + e];
        dst[i] = accumulate ? dst[i] + v : v;
      }
    }
  }
}

// traces of the interleaved field in sV (this lane's column) -> interleaved sT[(f*2+k)*NF + γ]
template <int P>
__device__ __forceinline__ void lane_traces_all(const double *sV, double *sT) {
  constexpr int NF = LDim<P>::NF;
  double t[2][NF];
  LaneOps<P>::template trace<0>(sV, t);
#pragma unroll
  for (int g = 0; g < NF; ++g) { sT[(0 * NF + g) * kLS] = t[0][g]; sT[(1 * NF + g) * kLS] = t[1][g]; }
  LaneOps<P>::template trace<1>(sV, t);
#pragma unroll
  for (int g = 0; g < NF; ++g) { sT[(2 * NF + g) * kLS] = t[0][g]; sT[(3 * NF + g) * kLS] = t[1][g]; }
  LaneOps<P>::template trace<2>(sV, t);
#pragma unroll
  for (int g = 0; g < NF; ++g) { sT[(4 * NF + g) * kLS] = t[0][g]; sT[(5 * NF + g) * kLS] = t[1][g]; }
  LaneOps<P>::template trace<3>(sV, t);
#pragma unroll
  for (int g = 0; g < NF; ++g) { sT[(6 * NF + g) * kLS] = t[0][g]; sT[(7 * NF + g) * kLS] = t[1][g]; }
}

// coalesced store of the interleaved traces of 32 elements to tr[e][8NF]
template <int NF>
__device__ __forceinline__ void lane_store_traces(double *__restrict__ tr, int64_t e0, int nel, const double *sT,
                                                  int lane) {
  double *dst = tr + e0 * 8 * NF;
  for (int i = lane; i < nel * 8 * NF; i += 32) {
    const int e = i / (8 * NF), r = i - e * 8 * NF;
    dst[i] = sT[r * kLS + e];
  }
}

template <int P, int F>
__device__ __forceinline__ void lane_face(const StageArgs &a, const double *trY, const double *sYl, double *sAl,
                                          int64_t e, const Geo &g, bool stageE, double sgn) {
  constexpr int NF = LDim<P>::NF;
  double t[2][NF];
  LaneOps<P>::template trace<F>(sYl, t);
  const int nb = a.nbr[4 * e + F];
  const int gf = a.nbrf[4 * e + F];
  double w = 0.5, k = 0.0;
  if (a.upwind) {
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
  const double mirrorY = stageE ? 1.0 : -1.0, mirrorX = stageE ? -1.0 : 1.0;
  const double sf = (F & 1) ? -1.0 : 1.0;
  const double *tn = nb >= 0 ? trY + ((int64_t)nb * 4 + gf) * 2 * NF : nullptr;
  double q[3][NF];
#pragma unroll
  for (int gm = 0; gm < NF; ++gm) {
    const double yn1 = nb >= 0 ? __ldg(tn + gm) : mirrorY * t[0][gm];
    const double yn2 = nb >= 0 ? __ldg(tn + NF + gm) : mirrorY * t[1][gm];
    const double d1 = w * (yn1 - t[0][gm]), d2 = w * (yn2 - t[1][gm]);
#pragma unroll
    for (int m = 0; m < 3; ++m) q[m][gm] = sf * (d1 * kLT2[F][m] - d2 * kLT1[F][m]);
  }
  if (a.upwind) {
    const double *to = a.trX + ((int64_t)e * 4 + F) * 2 * NF;
    const double *tx = nb >= 0 ? a.trX + ((int64_t)nb * 4 + gf) * 2 * NF : nullptr;
    const double *M = a.fmet + 12 * e + 3 * F;
    const double M0 = M[0], M1 = M[1], M2 = M[2];
    const double ps = (stageE ? 1.0 : -1.0) * sgn;
#pragma unroll
    for (int gm = 0; gm < NF; ++gm) {
      const double xo1 = __ldg(to + gm), xo2 = __ldg(to + NF + gm);
      const double xn1 = nb >= 0 ? __ldg(tx + gm) : mirrorX * xo1;
      const double xn2 = nb >= 0 ? __ldg(tx + NF + gm) : mirrorX * xo2;
      const double j1 = k * (xn1 - xo1), j2 = k * (xn2 - xo2);
      const double p1 = j1 * M0 + j2 * M1, p2 = j1 * M1 + j2 * M2;
#pragma unroll
      for (int m = 0; m < 3; ++m) q[m][gm] += ps * (p1 * kLT1[F][m] + p2 * kLT2[F][m]);
    }
  }
  LaneOps<P>::template lift<F>(q, sAl);
}

template <int P>
__global__ void __launch_bounds__(LDim<P>::WARPS * 32)
    lane_stage_kernel(StageArgs a, const double *__restrict__ trY, double *__restrict__ trOut) {
  using D = LDim<P>;
  constexpr int N = D::N, NF = D::NF, LD = D::LD;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *sY = smem + warp * D::WS;
  double *sA = sY + D::SY * kLS;
  const int64_t cs = a.n_tet * LD;
  const bool stageE = a.stage == STAGE_E;
  for (int64_t e0 = ((int64_t)blockIdx.x * D::WARPS + warp) * 32; e0 < a.n_tet;
       e0 += (int64_t)gridDim.x * D::WARPS * 32) {
    const int nel = (int)(a.n_tet - e0 < 32 ? a.n_tet - e0 : 32);
    const bool active = lane < nel;
    const int64_t e = e0 + lane;
    lane_load<N, LD>(a.Y, e0, nel, cs, sY, lane);
    __syncwarp();
    double *sYl = sY + lane, *sAl = sA + lane;
    if (a.do_curl) {
      LaneOps<P>::curl(sYl, sAl);
    } else {
#pragma unroll 4
      for (int i = 0; i < 3 * N; ++i) sAl[i * kLS] = 0.0;
    }
    if (a.do_flux && active) {
      const Geo g = a.geo[e];
      const double sgn = g.detF > 0 ? 1.0 : -1.0;
      lane_face<P, 0>(a, trY, sYl, sAl, e, g, stageE, sgn);
      lane_face<P, 1>(a, trY, sYl, sAl, e, g, stageE, sgn);
      lane_face<P, 2>(a, trY, sYl, sAl, e, g, stageE, sgn);
      lane_face<P, 3>(a, trY, sYl, sAl, e, g, stageE, sgn);
    }
    __syncwarp();
    // S2 + S6: inverse mass with geometry; the sY area now stages X (or dX)
    const bool upd = a.out_mode == OUT_UPDATE;
    if (upd) lane_load<N, LD>(a.X, e0, nel, cs, sY, lane);
    __syncwarp();
    if (active) {
      const Geo g = a.geo[e];
      const double cm = stageE ? g.inv_eps : -g.inv_mu;
      const double sc = upd ? a.dt * cm : cm;
      for (int b = 0; b < N; ++b) {
        const double v0 = sAl[b * kLS], v1 = sAl[(N + b) * kLS], v2 = sAl[(2 * N + b) * kLS];
        const double x0 = sc * (g.g[0] * v0 + g.g[1] * v1 + g.g[2] * v2);
        const double x1 = sc * (g.g[1] * v0 + g.g[3] * v1 + g.g[4] * v2);
        const double x2 = sc * (g.g[2] * v0 + g.g[4] * v1 + g.g[5] * v2);
        if (upd) {
          sYl[b * kLS] += x0;
          sYl[(N + b) * kLS] += x1;
          sYl[(2 * N + b) * kLS] += x2;
        } else {
          sYl[b * kLS] = x0;
          sYl[(N + b) * kLS] = x1;
          sYl[(2 * N + b) * kLS] = x2;
        }
      }
    }
    __syncwarp();
    if (upd) {
      lane_store<N, LD>(a.X, e0, nel, cs, sY, lane, false);
      if (trOut) {
        // traces of the updated field for the next stage's neighbours
        lane_traces_all<P>(sYl, sAl);
        __syncwarp();
        lane_store_traces<NF>(trOut, e0, nel, sA, lane);
      }
    } else {
      lane_store<N, LD>(a.dX, e0, nel, cs, sY, lane, a.out_mode == OUT_ACCUM);
    }
    __syncwarp();
  }
}

template <int P>
__global__ void __launch_bounds__(LDim<P>::WARPS * 32)
    lane_trace_kernel(const double *__restrict__ X, double *__restrict__ tr, int64_t n_tet) {
  using D = LDim<P>;
  constexpr int N = D::N, NF = D::NF, LD = D::LD;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *sY = smem + warp * D::WS;
  double *sA = sY + D::SY * kLS;
  const int64_t cs = n_tet * LD;
  for (int64_t e0 = ((int64_t)blockIdx.x * D::WARPS + warp) * 32; e0 < n_tet; e0 += (int64_t)gridDim.x * D::WARPS * 32) {
    const int nel = (int)(n_tet - e0 < 32 ? n_tet - e0 : 32);
    lane_load<N, LD>(X, e0, nel, cs, sY, lane);
    __syncwarp();
    lane_traces_all<P>(sY + lane, sA + lane);
    __syncwarp();
    lane_store_traces<NF>(tr, e0, nel, sA, lane);
    __syncwarp();
  }
}

template <int P>
static dgm_status lane_stage_p(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st) {
  using D = LDim<P>;
  const size_t smem = sizeof(double) * D::WS * D::WARPS;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(lane_stage_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_stage_kernel<P>, D::WARPS * 32, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t groups = (c->n_tet + 31) / 32;
  int64_t grid = (groups + D::WARPS - 1) / D::WARPS;
  if (grid > (int64_t)c->sms * occ) grid = (int64_t)c->sms * occ;
  lane_stage_kernel<P><<<(unsigned)grid, D::WARPS * 32, smem, st>>>(a, trY, trOut);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(c, DGM_ECUDA, std::string("lane_stage_kernel: ") + cudaGetErrorString(e));
  return DGM_OK;
}

template <int P>
static dgm_status lane_trace_p(dgm_ctx *c, const double *X, double *tr, cudaStream_t st) {
  using D = LDim<P>;
  const size_t smem = sizeof(double) * D::WS * D::WARPS;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(lane_trace_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lane_trace_kernel<P>, D::WARPS * 32, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t groups = (c->n_tet + 31) / 32;
  int64_t grid = (groups + D::WARPS - 1) / D::WARPS;
  if (grid > (int64_t)c->sms * occ) grid = (int64_t)c->sms * occ;
  lane_trace_kernel<P><<<(unsigned)grid, D::WARPS * 32, smem, st>>>(X, tr, c->n_tet);
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
  a.do_curl = do_curl;
  a.do_flux = do_flux;
  a.out_mode = out_mode;
  switch (c->p) {
    case 1: return lane_stage_p<1>(c, a, trY, trOut, st);
    case 2: return lane_stage_p<2>(c, a, trY, trOut, st);
    case 3: return lane_stage_p<3>(c, a, trY, trOut, st);
    case 4: return lane_stage_p<4>(c, a, trY, trOut, st);
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
  }
  return DGM_EORDER;
}

}  // namespace dgm
