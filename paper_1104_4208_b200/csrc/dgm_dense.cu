// Dense-contraction stage engine (FP64 tensor cores, mma.sync m8n8k4), sm_100a.
//
// The per-element operator is linear in the reference frame:
//   acc_T = Ĉ Ŷ_T + Σ_f L_f (A_f, B_f)_T,   Ẋ_T = ±(1/m_T) G'_T acc_T,
//   traces_T = Tr X_T,
// with Ĉ the reference curl, L_f the lift and Tr the tangential
// face traces.  Ĉ, L, Tr are the SAME matrices for every element,
// so applied to a tile of elements they are GEMMs: M = elements, N = output modes,
// K = input modes.  The matrices are assembled once per context from the exact
// recurrence / staged-trace programs (dgm_host.cpp: dense_build), so this engine
// computes the same operator as the sparse kernels with a different summation order.
//
// Why: the sparse recurrence path needs ~10x fewer flops, but every FMA of it reads
// its operand from shared memory (no register reuse), which caps it near 5-10 % of
// the FP64 pipe at p >= 7 (profiles/).  A register-blocked DMMA GEMM re-uses each
// operand from registers 6-8 times.  NORTH_STAR allows tensor cores where a dense
// contraction is measured to beat the sparse path; bench.py reports which engine ran.
//
// Per stage (E or H), three launches:
//   dense_flux_kernel   A, B face fields from the trace buffers (central/upwind/
//                       stabilised, PEC mirror), AB[e][(f*2+{A,B})*NF + γ]
//   gemm<EPI_STAGE>     acc = [Ŷ | AB] · B1, epilogue G'-mix, ±1/m, X += dt Ẋ (or write)
//   gemm<EPI_TRACE>     traces of the updated X = X · B2 -> trace buffer tr[e][f][k][γ]
#include <cstdint>
#include <cstdlib>
#include <string>

#include "dgm_internal.h"

namespace dgm {
namespace {

constexpr int BN = 96, BK = 16;  // BN: one warp column = three 32-column blocks
constexpr int WM = 16;             // warp tile: 16 rows x 96 columns (2 x 12 MMAs of 8x8)
constexpr int AKS = BK + 4;        // A tile row stride ([m][k] layout)

// CTA shape: BM elements x BNT columns; (BM/16) x NH warps.  Warps of one warp column
// see the same operator block mask.
template <int BM_, int NST_, int NH_>
struct Cfg {
  static constexpr int NH = NH_, BNT = BN * NH_, BST = BN * NH_ + 4;   // padded (conflict-free fragment loads)
  static constexpr int BM = BM_, NSTAGE = NST_, NTHREADS = (BM_ / WM) * NH_ * 32;
  static constexpr int MINB = NH_ == 1 ? (BM_ == 32 ? 4 : (BM_ == 64 ? 3 : 1)) : (BM_ == 64 ? 2 : 1);
  struct Smem {
    double A[NST_][BM_][AKS];
    double B[NST_][BK][BN * NH_ + 4];
  };
  static constexpr size_t EPI_BYTES = sizeof(double) * (BM_ * (BN * NH_ + 4) + BM_ * 8);   // C tile + geometry
  static constexpr size_t SMEM_DATA = sizeof(Smem) > EPI_BYTES ? sizeof(Smem) : EPI_BYTES;
  static constexpr size_t SMEM = SMEM_DATA + 8 * NST_ + 8;   // + one mbarrier per stage (B tile), next tile
};

enum { EPI_STAGE = 0, EPI_TRACE = 1 };

struct GemmArgs {
  // A operand, element e, column k (component-blocked rows, see DenseOps; every
  // 16-row k-tile lies inside one block):
  //   k <  k1: c = k / Nk, β = k % Nk  -> p0 + e*ld0 + c*cs + β       (β < N, else 0)
  //   k >= k1: j = (k-k1) / NFk, γ = ..  -> p1 + e*ld1 + j*NFk + γ    (γ < NF, else 0)
  const double *p0, *p1;
  int64_t ld0, ld1, cs;
  int k1, Nk, NFk;
  // k-tile geometry: k-tiles per A block below / above k1 (and float reciprocals)
  int k1t, nkA, nkF;
  float rnkA, rnkF;
  // B operand: pre-tiled pool [ntiles_n][nkt][BK][BST] (host: dense_build, `pool`),
  // columns as `tile_col` there: EPI_STAGE gathers the three component blocks of the
  // tile's 32 NH modes (warp columns alternate 8-mode groups); EPI_TRACE takes
  // contiguous columns (warp columns alternate 8-column groups)
  const double *Bm;
  int nkt;
  int NC;
  int Np;                  // operator columns per component (EPI_STAGE: column m*Np + β)
  const uint64_t *ktl;     // per non-zero k-tile: kt | (12-bit mask of non-zero 16x8 column groups per
                           // warp column, warp column h at bit 12h) << 16
  const int32_t *ktoff;
  int ntiles_n;
  int64_t n_tet;
  int Na;                  // valid rows per A block (k < k1): N, or Q for point values
  // epilogue
  int N, NF, LD;
  int ncols;   // valid output columns (EPI_TRACE: 8NF)
  const Geo *geo;
  double *X, *dX, *tr;
  double dt;
  int stageE, out_mode;
  // variable materials (reverse numerical integration): EPI_TRACE scales column
  // c*sQ + i by scale[e*sQ + i]; EPI_STAGE with raw != null writes the residual
  // v_c(β) to raw[e*rawld + c*rawNk + β] instead of updating; unit_m: cm = ±1
  const double *scale;
  int sQ;
  double *raw;
  int rawld, rawNk;
  int unit_m;
  int no_geo;   // EPI_STAGE: no G' mix (curved elements: the per-point factors carried it)
  unsigned long long *tile_ctr;   // dynamic tile counter [claims, arrivals] (self-resetting), or null: static order
  // EPI_STAGE, hybrid engine: the curl ĉ from the streamed sweeps is added to the
  // accumulator, ĉ[c][e][b] at cc + c*ccs + e*ldc + b for b < ncc (else 0)
  const double *cc;
  int64_t ccs;
  int ldc, ncc;
};

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
// 16-byte async copy, zero-filling beyond `bytes` (0, 8 or 16)
__device__ __forceinline__ void cpa16z(double *dst, const double *src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(su32(dst)), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cpa16(double *dst, const double *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NW>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NW) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "MBW_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra MBW_DONE;\n\t"
      "bra MBW_LOOP;\n\t"
      "MBW_DONE:\n\t}\n" ::"r"(su32(m)),
      "r"(parity)
      : "memory");
}
// one bulk copy global -> shared (the B tile), completion counted on the mbarrier
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *m) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(m))
               : "memory");
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// the 8-column groups j0 + j of one k-tile for the set bits j of M: k4 outermost, so
// the DMMAs of one k4 step are independent (hides the DMMA dependency latency)
template <unsigned M, int BST>
__device__ __forceinline__ void mma_set(double (&acc)[12][2][2], const double (&a)[BK / 4][2], const double *bw,
                                        int j0) {
#pragma unroll
  for (int k4 = 0; k4 < BK / 4; ++k4) {
    double b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (M >> j & 1u) b[j] = bw[k4 * 4 * BST + (j0 + j) * 8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (M >> j & 1u)
#pragma unroll
        for (int i = 0; i < 2; ++i) dmma(acc[j0 + j][i][0], acc[j0 + j][i][1], a[k4][i], b[j]);
  }
}

// load k-tile kt of A ([m][k], 16-byte copies of mode pairs) and B into stage st.
// Thread tid copies A rows tid/8 + i NTHREADS/8 at mode pair tid%8 (the same pair for
// every row), so per k-tile only the block base and the zero-fill bound are recomputed.
// B comes from the pre-tiled pool (one [BK][BST] tile per (n-tile, k-tile), already
// in the shared-memory layout): one bulk copy by thread 0 on the stage's mbarrier.
// per-tile part of a thread's A addressing: row offsets of its first row in both
// A blocks, and how many of its rows exist (ragged last tile)
struct ARow {
  int64_t off0, off1;
  int nrow;
};

template <int EPI, class C>
__device__ __forceinline__ void load_tile(const GemmArgs &g, typename C::Smem &sm, uint64_t *mbar, int st, const ARow &ar,
                                          int nt, int kt, int tid) {
  constexpr int BM = C::BM, NTHREADS = C::NTHREADS, BST = C::BST;
  constexpr int RSTEP = NTHREADS / 8;   // rows between one thread's A copies
  const bool lo = kt < g.k1t;
  // block index and first in-block row of the tile: small exact quotients by float
  // reciprocal ((kt + 0.5)/n is at least 0.5/n away from an integer)
  const int kr = lo ? kt : kt - g.k1t;
  const int blk = (int)(((float)kr + 0.5f) * (lo ? g.rnkA : g.rnkF));
  const int q0 = (kr - blk * (lo ? g.nkA : g.nkF)) * BK;
  const int lim = lo ? g.Na : g.NF;
  const int kp = tid & 7;
  const int q = q0 + 2 * kp;
  const int bq = q + 1 < lim ? 16 : (q < lim ? 8 : 0);
  const double *src = lo ? g.p0 + blk * g.cs + ar.off0 + q : g.p1 + (int64_t)blk * g.NFk + ar.off1 + q;
  const int64_t rs = RSTEP * (lo ? g.ld0 : g.ld1);
  double *dst = &sm.A[st][tid >> 3][2 * kp];
#pragma unroll
  for (int i = 0; i < BM / RSTEP; ++i) {
    // zero-size copies read nothing (zero fill), so the pointer of a missing row is not used
    cpa16z(dst + i * RSTEP * AKS, src, i * RSTEP < ar.nrow ? bq : 0);
    src += rs;
  }
  if (tid == 0)
    bulk_load(&sm.B[st][0][0], g.Bm + ((int64_t)nt * g.nkt + kt) * (BK * BST), BK * BST * sizeof(double), &mbar[st]);
}

template <int EPI, class C>
__global__ void __launch_bounds__(C::NTHREADS, C::MINB) gemm_kernel(GemmArgs g) {
  constexpr int BM = C::BM, NSTAGE = C::NSTAGE, NTHREADS = C::NTHREADS, NH = C::NH, BNT = C::BNT, BST = C::BST;
  extern __shared__ __align__(16) unsigned char dsm[];
  typename C::Smem &sm = *reinterpret_cast<typename C::Smem *>(dsm);
  uint64_t *mbar = reinterpret_cast<uint64_t *>(dsm + C::SMEM_DATA);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&mbar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned ph = 0;   // bit s: parity of the next completion of stage s's B tile
  const int wm = warp % (BM / WM), wn = warp / (BM / WM);
  const int gr = lane >> 2, gc = lane & 3;   // fragment row / k index
  const int64_t mtiles = (g.n_tet + BM - 1) / BM;
  const int64_t ntile_total = mtiles * g.ntiles_n;
  // dynamic tile order: CTAs take tiles in sequence from a counter (zeroed by the last
  // CTA of the previous launch), so the n-tiles of one m-tile start together and share its A rows in L2
  long long *tnext = reinterpret_cast<long long *>(dsm + C::SMEM_DATA + 8 * NSTAGE);
  for (int64_t t = blockIdx.x; t < ntile_total;) {
    const int64_t m0 = (t / g.ntiles_n) * BM;
    const int nt = (int)(t % g.ntiles_n);
    const int n0 = nt * BNT;
    const uint64_t *kts = g.ktl + g.ktoff[nt];
    const int nk = g.ktoff[nt + 1] - g.ktoff[nt];
    double acc[12][2][2];   // [column group j][row group i][pair]
#pragma unroll
    for (int j = 0; j < 12; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) acc[j][i][0] = acc[j][i][1] = 0.0;
    if (EPI == EPI_STAGE && g.out_mode == OUT_UPDATE) {
      // pull this tile's X block (64 elements x 3 x 32 modes) into L2 while the k-loop
      // runs, so the read-modify-write epilogue does not wait on HBM
      const int64_t cs = g.n_tet * g.LD;
      for (int q = tid; q < BM * 3; q += NTHREADS) {
        const int64_t e = m0 + q / 3;
        if (e < g.n_tet) {
          const double *px = g.X + (q % 3) * cs + e * g.LD + 32 * NH * nt;
#pragma unroll
          for (int l = 0; l < 2 * NH; ++l) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(px + 16 * l));
          if (g.cc && 32 * NH * nt < g.ncc) {   // hybrid: the tile's block of the sweeps' ĉ too
            const double *pc = g.cc + (q % 3) * g.ccs + e * g.ldc + 32 * NH * nt;
#pragma unroll
            for (int l = 0; l < 2 * NH; ++l) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pc + 16 * l));
          }
        }
      }
    }
    ARow ar;
    {
      const int64_t eA = m0 + (tid >> 3);
      ar.off0 = eA * g.ld0;
      ar.off1 = eA * g.ld1;
      const int64_t nr = g.n_tet - eA;
      ar.nrow = nr > BM ? BM : (int)nr;
    }
    // prologue
#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
      if (s < nk) load_tile<EPI, C>(g, sm, mbar, s, ar, nt, (int)(kts[s] & 0xFFFFu), tid);
      cp_commit();
    }
    uint64_t kcur = nk > 0 ? kts[0] : 0ull;
    for (int it = 0; it < nk; ++it) {
      const uint64_t knext = it + 1 < nk ? kts[it + 1] : 0ull;   // one ahead: off the critical path
      const int st = it % NSTAGE;
      cp_wait<NSTAGE - 2>();
      mbar_wait(&mbar[st], (ph >> st) & 1u);
      ph ^= 1u << st;
      __syncthreads();
      const int nx = it + NSTAGE - 1;
      if (nx < nk) load_tile<EPI, C>(g, sm, mbar, nx % NSTAGE, ar, nt, (int)(kts[nx] & 0xFFFFu), tid);
      cp_commit();
      double a[BK / 4][2];
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4)
#pragma unroll
        for (int i = 0; i < 2; ++i) a[k4][i] = sm.A[st][wm * WM + i * 8 + gr][k4 * 4 + gc];
      const unsigned m12 = (unsigned)(kcur >> (16 + 12 * wn)) & 0xFFFu;   // this warp column's non-zero 16x8 groups
      kcur = knext;
      // skip zero operator blocks: per 32-column block a warp-uniform switch over its
      // mask of non-zero 8-column groups (whole 16-row k-tiles, so the tensor pipe is not
      // occupied); the non-zero groups run interleaved with k4 outermost, so
      // consecutive DMMAs accumulate into different registers
      const double *bw = &sm.B[st][gc][wn * BN + gr];
#pragma unroll
      for (int grp = 0; grp < 3; ++grp) {
        switch ((m12 >> (4 * grp)) & 0xFu) {
#define DGM_SET(M) \
  case M: mma_set<M, BST>(acc, a, bw, grp * 4); break;
          DGM_SET(1) DGM_SET(2) DGM_SET(3) DGM_SET(4) DGM_SET(5) DGM_SET(6) DGM_SET(7) DGM_SET(8)
          DGM_SET(9) DGM_SET(10) DGM_SET(11) DGM_SET(12) DGM_SET(13) DGM_SET(14) DGM_SET(15)
#undef DGM_SET
          default: break;
        }
      }
    }
    cp_wait<0>();
    __syncthreads();
    if (EPI == EPI_TRACE) {
      // C fragment: row gr (+8i), cols 2gc, 2gc+1 (+8j) -> tr[e][col]
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int64_t e = m0 + wm * WM + i * 8 + gr;
        if (e >= g.n_tet) continue;
        double *row = g.tr + e * (int64_t)g.ncols;
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          const int col = n0 + (j * NH + wn) * 8 + 2 * gc;   // warp columns alternate 8-column groups
          double v0 = acc[j][i][0], v1 = acc[j][i][1];
          if (g.scale) {   // point values: quadrature weight / material at the point
            const double *sc = g.scale + e * g.sQ;
            v0 *= col < g.ncols ? sc[col % g.sQ] : 0.0;
            v1 *= col + 1 < g.ncols ? sc[(col + 1) % g.sQ] : 0.0;
          }
          if (col + 1 < g.ncols) {
            *reinterpret_cast<double2 *>(row + col) = make_double2(v0, v1);
          } else if (col < g.ncols) {
            row[col] = v0;
          }
        }
      }
    } else {
      // stage the tile in shared memory, then per (element, mode): G' mix and update
      double(*Cs)[BST] = reinterpret_cast<double(*)[BST]>(dsm);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          const int r = wm * WM + i * 8 + gr, c = wn * BN + j * 8 + 2 * gc;
          Cs[r][c] = acc[j][i][0];
          Cs[r][c + 1] = acc[j][i][1];
        }
      // per-element geometry rows after the tile: G' (6), ±1/m
      double(*Gs)[8] = reinterpret_cast<double(*)[8]>(dsm + sizeof(double) * BM * BST);
      for (int r = tid; r < BM; r += NTHREADS) {
        const int64_t e = m0 + r;
        if (e < g.n_tet) {
          const Geo &G = g.geo[e];
#pragma unroll
          for (int q = 0; q < 6; ++q) Gs[r][q] = G.g[q];
          Gs[r][6] = g.unit_m ? (g.stageE ? 1.0 : -1.0) : (g.stageE ? G.inv_eps : -G.inv_mu);
        }
      }
      __syncthreads();
      constexpr int MODES = BNT / 3;   // 32 NH modes; the warp columns alternate 8-mode groups
      constexpr int U = 4;   // items per batch: their 3U loads are in flight together
      const int64_t cs = g.n_tet * g.LD;
      const bool upd = g.out_mode == OUT_UPDATE;
      double *out = upd ? g.X : g.dX;
      for (int base = tid; base < BM * MODES; base += U * NTHREADS) {
        int64_t o[U];
        double xv[U][3], cv[U][3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * NTHREADS;
          const int r = idx / MODES, ml = idx - r * MODES;
          const int64_t e = m0 + r;
          const int b = 32 * NH * nt + ml;
          o[u] = (idx < BM * MODES && e < g.n_tet && b < g.N) ? e * g.LD + b : -1;
#pragma unroll
          for (int cc = 0; cc < 3; ++cc)
            xv[u][cc] = (o[u] >= 0 && g.out_mode != OUT_WRITE && !g.raw) ? out[cc * cs + o[u]] : 0.0;
          const bool hc = g.cc && o[u] >= 0 && b < g.ncc;
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) cv[u][cc] = hc ? g.cc[cc * g.ccs + e * g.ldc + b] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (o[u] < 0) continue;
          const int idx = base + u * NTHREADS;
          const int r = idx / MODES, ml = idx - r * MODES;
          const double *G = Gs[r];
          const double cm = G[6];
          // tile mode ml -> warp column h = (ml/8) % NH, its mode ((ml/8)/NH) 8 + ml%8
          const int hb = ((ml >> 3) % NH) * BN + ((ml >> 3) / NH) * 8 + (ml & 7);
          const double v0 = Cs[r][hb] + cv[u][0], v1 = Cs[r][32 + hb] + cv[u][1], v2 = Cs[r][64 + hb] + cv[u][2];
          if (g.raw) {   // residual before the (variable-material) inverse mass
            double *rw = g.raw + (m0 + r) * (int64_t)g.rawld + 32 * NH * nt + ml;
            rw[0] = v0;
            rw[g.rawNk] = v1;
            rw[2 * g.rawNk] = v2;
            continue;
          }
          const double x0 = g.no_geo ? cm * v0 : cm * (G[0] * v0 + G[1] * v1 + G[2] * v2);
          const double x1 = g.no_geo ? cm * v1 : cm * (G[1] * v0 + G[3] * v1 + G[4] * v2);
          const double x2 = g.no_geo ? cm * v2 : cm * (G[2] * v0 + G[4] * v1 + G[5] * v2);
          const double sc = upd ? g.dt : 1.0;
          out[o[u]] = xv[u][0] + sc * x0;
          out[cs + o[u]] = xv[u][1] + sc * x1;
          out[2 * cs + o[u]] = xv[u][2] + sc * x2;
        }
      }
    }
    if (tid == 0) *tnext = g.tile_ctr ? (long long)atomicAdd(g.tile_ctr, 1ull) + gridDim.x : t + gridDim.x;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // epilogue writes before the next bulk copies
    __syncthreads();
    t = *tnext;
    __syncthreads();
  }
  // self-resetting tile counter: the last CTA to finish zeroes it for the next launch
  // (every CTA's claims on ctr[0] precede its arrival on ctr[1])
  if (g.tile_ctr && tid == 0) {
    __threadfence();
    if (atomicAdd(g.tile_ctr + 1, 1ull) == (unsigned long long)gridDim.x - 1ull) {
      g.tile_ctr[0] = 0ull;
      g.tile_ctr[1] = 0ull;
      __threadfence();
    }
  }
}

// A, B face fields of every (element, face, mode) from the trace buffers
// (tr[e][f][k][γ]); same flux as the stage kernels (reading G1/G2/G17).
template <bool UP>
__global__ void dense_flux_kernel(StageArgs a, const double *__restrict__ trY, double *__restrict__ AB, int NF,
                                  int NFk) {
  const int64_t total = a.n_tet * 4 * NF;
  const bool stageE = a.stage == STAGE_E;
  const double mirrorY = stageE ? 1.0 : -1.0, mirrorX = stageE ? -1.0 : 1.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ef = i / NF;
    const int gm = (int)(i - ef * NF);
    const int64_t e = ef >> 2;
    const int f = (int)(ef & 3);
    const int nb = a.nbr[ef];
    const int gf = a.nbrf[ef];
    double w = 0.5, kk = 0.0;
    if (UP) {
      const double Zm = a.geo[e].Z, Zp = nb >= 0 ? a.geo[nb].Z : Zm;
      if (stageE) {
        w = Zp / (Zm + Zp);
        kk = 1.0 / (Zm + Zp);
      } else {
        const double Ym = 1.0 / Zm, Yp = 1.0 / Zp;
        w = Yp / (Ym + Yp);
        kk = 1.0 / (Ym + Yp);
      }
    }
    const double sf = (f & 1) ? -1.0 : 1.0;
    const double *to = trY + ef * 2 * NF;
    const double o1 = __ldg(to + gm), o2 = __ldg(to + NF + gm);
    double n1, n2;
    if (nb >= 0) {
      const double *tn = trY + ((int64_t)nb * 4 + gf) * 2 * NF;
      n1 = __ldg(tn + gm);
      n2 = __ldg(tn + NF + gm);
    } else {
      n1 = mirrorY * o1;
      n2 = mirrorY * o2;
    }
    double h1 = 0.0, h2 = 0.0;   // stabilised flux (E stage): Δ_k -= H^F_k
    if (a.HF) {
      const double *hf = a.HF + (int64_t)a.fid[ef] * 2 * NF;
      h1 = __ldg(hf + gm);
      h2 = __ldg(hf + NF + gm);
    }
    double A = -sf * (w * (n2 - o2) - h2), B = sf * (w * (n1 - o1) - h1);
    if (UP) {
      const double *xo = a.trX + ef * 2 * NF;
      const double xo1 = __ldg(xo + gm), xo2 = __ldg(xo + NF + gm);
      double xn1, xn2;
      if (nb >= 0) {
        const double *xn = a.trX + ((int64_t)nb * 4 + gf) * 2 * NF;
        xn1 = __ldg(xn + gm);
        xn2 = __ldg(xn + NF + gm);
      } else {
        xn1 = mirrorX * xo1;
        xn2 = mirrorX * xo2;
      }
      const double j1 = kk * (xn1 - xo1), j2 = kk * (xn2 - xo2);
      const double *M = a.fmet + 12 * e + 3 * f;
      const double ps = (stageE ? 1.0 : -1.0) * (a.geo[e].detF > 0 ? 1.0 : -1.0);
      A += ps * (j1 * M[0] + j2 * M[1]);
      B += ps * (j1 * M[1] + j2 * M[2]);
    }
    double *o = AB + ef * 2 * NFk;   // AB[e][(f*2+{A,B})*NFk + γ]
    o[gm] = A;
    o[NFk + gm] = B;
  }
}

template <int EPI, class C>
dgm_status gemm_go_c(dgm_ctx *c, const GemmArgs &g0, cudaStream_t st) {
  GemmArgs g = g0;
  g.tile_ctr = c->dense.tile_ctr;
  g.k1t = g.k1 / BK;
  g.nkA = g.Nk / BK;
  g.nkF = g.NFk / BK;
  g.rnkA = 1.0f / (float)g.nkA;
  g.rnkF = 1.0f / (float)g.nkF;
  const size_t smem = C::SMEM;
  auto kern = gemm_kernel<EPI, C>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NTHREADS, smem);
  if (occ < 1) occ = 1;
  const int64_t tiles = (g.n_tet + C::BM - 1) / C::BM * g.ntiles_n;
  int64_t grid = (int64_t)c->sms * occ;
  if (grid > tiles) grid = tiles;
  kern<<<(unsigned)grid, C::NTHREADS, smem, st>>>(g);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("gemm_kernel: ") + cudaGetErrorString(e));
}

// CTA tile configuration (measurement overrides): DGM_DENSE_CFG for every GEMM,
// DGM_STAGE_CFG / DGM_TRACE_CFG per GEMM type (0: 64x3 stages, the default; 1: 64x4;
// 2: 128x3; 3: 32x4)
int dense_cfg(int epi) {
  const char *v = std::getenv(epi == EPI_STAGE ? "DGM_STAGE_CFG" : "DGM_TRACE_CFG");
  if (!(v && *v)) v = std::getenv("DGM_DENSE_CFG");
  return v && *v ? std::atoi(v) : 0;
}

template <int EPI, int NHV>
dgm_status gemm_go_nh(dgm_ctx *c, const GemmArgs &g, cudaStream_t st) {
  switch (dense_cfg(EPI)) {
    case 1: return gemm_go_c<EPI, Cfg<64, 4, NHV>>(c, g, st);
    case 2: return gemm_go_c<EPI, Cfg<128, 3, NHV>>(c, g, st);
    case 3: return gemm_go_c<EPI, Cfg<32, 4, NHV>>(c, g, st);
    default: return gemm_go_c<EPI, Cfg<64, 3, NHV>>(c, g, st);
  }
}

// stage GEMMs: one warp column (gathered component blocks); trace-type GEMMs: the
// context's choice (two warp columns halve the A re-reads at p >= 8)
template <int EPI>
dgm_status gemm_go(dgm_ctx *c, const GemmArgs &g, cudaStream_t st) {
  if ((EPI == EPI_TRACE ? c->dense.trace_nh : c->dense.stage_nh) == 2) return gemm_go_nh<EPI, 2>(c, g, st);
  return gemm_go_nh<EPI, 1>(c, g, st);
}

}  // namespace

dgm_status launch_dense_stage(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st) {
  const DenseOps &D = c->dense;
  const int v = a.stage == STAGE_E ? 0 : 1;   // updated field: operator variant (mixed orders)
  if (a.do_flux) {
    const int64_t total = a.n_tet * 4 * c->NF;
    int64_t grid = (total + 255) / 256;
    if (grid > 16 * (int64_t)c->sms) grid = 16 * (int64_t)c->sms;
    if (a.upwind)
      dense_flux_kernel<true><<<(unsigned)grid, 256, 0, st>>>(a, trY, D.AB, c->NF, (c->NF + BK - 1) / BK * BK);
    else
      dense_flux_kernel<false><<<(unsigned)grid, 256, 0, st>>>(a, trY, D.AB, c->NF, (c->NF + BK - 1) / BK * BK);
    c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(c, DGM_ECUDA, std::string("dense_flux_kernel: ") + cudaGetErrorString(e));
  }
  GemmArgs g{};
  g.p0 = a.Y;
  g.p1 = D.AB;
  g.ld0 = c->LD;
  g.ld1 = 8 * ((c->NF + BK - 1) / BK * BK);
  g.cs = c->n_tet * c->LD;
  g.k1 = D.k1a;
  g.Nk = D.k1a / 3;
  g.NFk = (c->NF + BK - 1) / BK * BK;
  g.Bm = D.B1[v];
  g.nkt = D.nkt1;
  g.NC = D.nc1;
  g.Np = D.nc1 / 3;
  // curl only / flux only: restrict the k-tile lists.  Hybrid engine: the curl comes
  // from the streamed recurrence sweeps (ĉ, added in the epilogue), the GEMM does the
  // lift only
  int sel = (a.do_curl ? 1 : 0) | (a.do_flux ? 2 : 0);
  if (c->sparse_curl && a.do_curl) {
    dgm_status s = launch_curl(c, a.Y, D.Cc, st);
    if (s != DGM_OK) return s;
    sel &= 2;
    g.cc = D.Cc;
    g.ccs = c->n_tet * (int64_t)D.ldc;
    g.ldc = D.ldc;
    g.ncc = c->p * (c->p + 1) * (c->p + 2) / 6;
  }
  g.ktl = D.ktl1[v][sel];
  g.ktoff = D.ktoff1[v][sel];
  g.ntiles_n = D.nc1 / 3 / (32 * D.stage_nh);
  g.n_tet = c->n_tet;
  g.N = c->N;
  g.NF = c->NF;
  g.LD = c->LD;
  g.ncols = 3 * c->N;
  g.geo = c->d_geo;
  g.X = a.X;
  g.dX = a.dX;
  g.dt = a.dt;
  g.stageE = a.stage == STAGE_E;
  g.out_mode = a.out_mode;
  g.Na = c->N;
  if (c->matq) {
    // variable materials: write the residual, then the reverse-numerical-integration
    // inverse mass as two more GEMMs: residual -> point values ×
    // ŵ_i/m(x_i), point values -> modes (1/‖φ‖²), then G' and the update
    const int Nk = D.k1a / 3, Qk = c->Qk;
    g.raw = D.AC;
    g.rawld = 3 * Nk;
    g.rawNk = Nk;
    dgm_status s = gemm_go<EPI_STAGE>(c, g, st);
    if (s != DGM_OK) return s;
    if (D.use_sumfact) {   // sum-factorised point transforms, O(p⁴)
      SumfactArgs sa{};
      sa.AC = D.AC;
      sa.acld = 3 * Nk;
      sa.acNk = Nk;
      sa.Pc = D.sf_tab + D.sf_pc;
      sa.Bb = D.sf_tab + D.sf_bb;
      sa.Ca = D.sf_tab + D.sf_ca;
      sa.inv_norms = D.sf_tab + D.sf_in;
      sa.modes = D.sf_modes;
      sa.pairs = D.sf_pairs;
      sa.K = c->curved ? (a.stage == STAGE_E ? D.KE : D.KH) : nullptr;
      sa.SW = a.stage == STAGE_E ? D.SWe : D.SWm;
      sa.Qk = Qk;
      sa.geo = c->d_geo;
      sa.X = a.X;
      sa.dX = a.dX;
      sa.dt = a.dt;
      sa.n_tet = c->n_tet;
      sa.LD = c->LD;
      sa.stageE = a.stage == STAGE_E;
      sa.out_mode = a.out_mode;
      if ((s = launch_sumfact(c, sa, st)) != DGM_OK) return s;
      if (a.out_mode == OUT_UPDATE && trOut) return launch_dense_traces(c, a.X, trOut, st, v);
      return DGM_OK;
    }
    GemmArgs f{};
    f.p0 = f.p1 = D.AC;
    f.ld0 = f.ld1 = 3 * Nk;
    f.cs = Nk;
    f.k1 = 1 << 30;
    f.Nk = Nk;
    f.NFk = Nk;
    f.Na = c->N;
    f.Bm = D.Bf;
    f.nkt = D.nktf;
    f.NC = D.ncf;
    f.ktl = D.ktlf;
    f.ktoff = D.ktofff;
    f.ntiles_n = D.ncf / (BN * D.trace_nh);
    f.n_tet = c->n_tet;
    f.ncols = 3 * Qk;
    f.tr = D.P;
    f.scale = c->curved ? nullptr : (a.stage == STAGE_E ? D.SWe : D.SWm);
    f.sQ = Qk;
    if ((s = gemm_go<EPI_TRACE>(c, f, st)) != DGM_OK) return s;
    // curved elements: the per-point 3x3 factor ŵ_i F(ξ_i)ᵀF(ξ_i)/(m det F(ξ_i)) replaces
    // ŵ_i/m(x_i) here and the element's G' after the back transform
    if (c->curved && (s = launch_pointmix(c, D.P, a.stage == STAGE_E ? D.KE : D.KH, st)) != DGM_OK) return s;
    GemmArgs b = g;
    b.raw = nullptr;
    b.cc = nullptr;   // ĉ entered the residual already
    b.p0 = b.p1 = D.P;
    b.ld0 = b.ld1 = 3 * Qk;
    b.cs = Qk;
    b.k1 = 1 << 30;
    b.Nk = Qk;
    b.NFk = Qk;
    b.Na = c->Q;
    b.Bm = D.Bb;
    b.nkt = D.nktb;
    b.ktl = D.ktlb;
    b.ktoff = D.ktoffb;
    b.unit_m = 1;
    b.no_geo = c->curved;
    if ((s = gemm_go<EPI_STAGE>(c, b, st)) != DGM_OK) return s;
  } else {
    dgm_status s = gemm_go<EPI_STAGE>(c, g, st);
    if (s != DGM_OK) return s;
  }
  if (a.out_mode == OUT_UPDATE && trOut) return launch_dense_traces(c, a.X, trOut, st, v);
  return DGM_OK;
}

namespace {
// curved elements: the 3x3 point factor of the approximate inverse
// mass on the point values of the residual, one thread per (element, point)
__global__ void pointmix_kernel(double *__restrict__ P, const double *__restrict__ K, int64_t n_tet, int Q, int Qk) {
  const int64_t total = n_tet * Q;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / Q;
    const int q = (int)(i - e * Q);
    double *pe = P + e * 3 * (int64_t)Qk + q;
    const double *k = K + (e * Qk + q) * 6;
    const double v0 = pe[0], v1 = pe[Qk], v2 = pe[2 * Qk];
    pe[0] = k[0] * v0 + k[1] * v1 + k[2] * v2;
    pe[Qk] = k[1] * v0 + k[3] * v1 + k[4] * v2;
    pe[2 * Qk] = k[2] * v0 + k[4] * v1 + k[5] * v2;
  }
}
}  // namespace

dgm_status launch_pointmix(dgm_ctx *c, double *P, const double *K, cudaStream_t st) {
  const int64_t total = c->n_tet * c->Q;
  int64_t grid = (total + 255) / 256;
  if (grid > 16 * (int64_t)c->sms) grid = 16 * (int64_t)c->sms;
  if (grid < 1) return DGM_OK;
  pointmix_kernel<<<(unsigned)grid, 256, 0, st>>>(P, K, c->n_tet, c->Q, c->Qk);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("pointmix_kernel: ") + cudaGetErrorString(e));
}

dgm_status launch_curl(dgm_ctx *c, const double *Y, double *C, cudaStream_t st) {
  switch (c->p) {
    case 4: return launch_curl_p4(c, Y, C, st);
    case 5: return launch_curl_p5(c, Y, C, st);
    case 6: return launch_curl_p6(c, Y, C, st);
    case 7: return launch_curl_p7(c, Y, C, st);
    case 8: return launch_curl_p8(c, Y, C, st);
    case 9: return launch_curl_p9(c, Y, C, st);
    case 10: return launch_curl_p10(c, Y, C, st);
  }
  return set_err(c, DGM_EORDER, "streamed curl sweeps: orders 4..10");
}

dgm_status launch_dense_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st, int field) {
  const DenseOps &D = c->dense;
  GemmArgs g{};
  g.p0 = X;
  g.p1 = X;
  g.ld0 = g.ld1 = c->LD;
  g.cs = c->n_tet * c->LD;
  g.k1 = 1 << 30;
  g.Nk = D.k1a / 3;
  g.NFk = (c->NF + BK - 1) / BK * BK;
  g.Na = c->N;
  g.Bm = D.B2[field];
  g.nkt = D.nkt2;
  g.NC = D.nc2;
  g.ktl = D.ktl2[field];
  g.ktoff = D.ktoff2[field];
  g.ntiles_n = D.nc2 / (BN * D.trace_nh);
  g.n_tet = c->n_tet;
  g.N = c->N;
  g.NF = c->NF;
  g.LD = c->LD;
  g.ncols = 8 * c->NF;
  g.tr = tr;
  return gemm_go<EPI_TRACE>(c, g, st);
}

}  // namespace dgm
