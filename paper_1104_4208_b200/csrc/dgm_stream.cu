// Streamed-table high-order stage kernels (p > kLanePmax), sm_100a FP64.
//
// The per-element algorithm of the sparse engine (as in the
// lane-pair kernels of dgm_lane.cu): recurrence curl, flux on the trace-buffer
// traces, staged sum-factorised lift, inverse mass with G'
// (PAPER.md:465-476), symplectic-Euler update, traces of the
// updated field.
//
// Execution shape.  One persistent CTA per SM.  Each warp owns KW elements at a
// time (interleaved in its own shared-memory workspace, slot v of element k at
// ws[v*KW + k]) and executes every program row for them, so all warps do identical
// work.  The program tables (curl, lifts, traces: ELL passes of {coef, src} terms)
// stream through a double-buffered shared-memory chunk ring: while the warps run
// chunk g from shared memory, one thread has a bulk TMA copy (cp.async.bulk +
// mbarrier complete_tx) of chunk g+1 in flight.  Term operands therefore come from
// shared memory instead of L1/L2 (the K=1 kernels were latency-bound on those
// loads), a DAG level needs only __syncwarp (the element is warp-private), and the
// only CTA barrier is the buffer hand-off once per chunk, with balanced work.
#include <cstdint>
#include <cstdlib>
#include <string>

#include "dgm_internal.h"

namespace dgm {
namespace {

__constant__ double sT1[4][3] = {{-1, 1, 0}, {0, 1, 0}, {1, 0, 0}, {1, 0, 0}};
__constant__ double sT2[4][3] = {{-1, 0, 1}, {0, 0, 1}, {0, 0, 1}, {0, 1, 0}};

template <int P>
struct DS {
  static constexpr int N = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NF = (P + 1) * (P + 2) / 2;
  static constexpr int LD = (N + 3) & ~3;
  static constexpr int ACC = 9 * N;              // curl accumulator slots (gen/plan.py)
  static constexpr int SAB = 12 * N;             // face fields (A, B) pairs
  static constexpr int SCR = (3 * N + 1) & ~1;   // staged trace/lift pair scratch (dead sweep region)
  static constexpr int WS = 12 * N + 2 * NF;
  static constexpr int GEO = 10;
};

template <int K>
__device__ __forceinline__ void ldk(const double *p, double (&v)[K]) {
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int j = 0; j < K / 2; ++j) {
      const double2 t = reinterpret_cast<const double2 *>(p)[j];
      v[2 * j] = t.x;
      v[2 * j + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = p[k];
  }
}

template <int K>
__device__ __forceinline__ void stk(double *p, const double (&v)[K]) {
  if constexpr (K % 2 == 0) {
#pragma unroll
    for (int j = 0; j < K / 2; ++j) reinterpret_cast<double2 *>(p)[j] = make_double2(v[2 * j], v[2 * j + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = v[k];
  }
}

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra WAIT_DONE;\n\t"
      "bra WAIT_LOOP;\n\t"
      "WAIT_DONE:\n\t}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
// one bulk TMA copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void tma_load(void *dst, const void *src, unsigned bytes, uint64_t *m) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}

extern __shared__ __align__(128) char smem_raw[];

// CTA-uniform chunk pipeline state.  Buffers are addressed from the shared-memory
// symbol itself (not a stored generic pointer) so the compiler emits LDS.
struct Pipe {
  int chunk_bytes;
  unsigned gc;   // chunks consumed so far
};
__device__ __forceinline__ uint64_t *pipe_mbar(int b) { return reinterpret_cast<uint64_t *>(smem_raw) + b; }
__device__ __forceinline__ char *pipe_buf(const Pipe &pp, int b) { return smem_raw + 128 + (size_t)b * pp.chunk_bytes; }

// Start chunk ci: barrier (everyone is done with the other buffer), thread 0 issues
// the next chunk of the schedule into it, then wait for chunk ci itself.
__device__ __forceinline__ const char *chunk_acquire(const DevStream &S, int ci, bool more, Pipe &pp, int tid) {
  __syncthreads();
  if (tid == 0) {
    int nci = ci + 1;
    bool go = true;
    if (nci == S.nchunk) {
      nci = 0;
      go = more;
    }
    if (go) {
      const StreamChunk c = S.chunks[nci];
      const int b = (pp.gc + 1) & 1;
      tma_load(pipe_buf(pp, b), S.base + c.off, c.bytes, pipe_mbar(b));
    }
  }
  mbar_wait(pipe_mbar(pp.gc & 1), (pp.gc >> 1) & 1);
  return pipe_buf(pp, pp.gc & 1);
}

// Run program pi for this warp's elements.  R supplies Acc, init(acc),
// term(acc, {coef, src}, level) and store(dst, acc).  Passes carry a uniform width
// (padded terms have coef 0), and two passes of the same level are interleaved so a
// lane has two independent rows in flight.
template <typename R>
__device__ __forceinline__ void run_prog(const DevStream &S, int pi, bool more, bool active, Pipe &pp, int tid,
                                         int lane, const R &r) {
  int lvl = 0;
  const int c0 = S.first[pi], c1 = c0 + S.count[pi];
  for (int ci = c0; ci < c1; ++ci) {
    const char *buf = chunk_acquire(S, ci, more, pp, tid);
    if (active) {
      const int np = S.chunks[ci].npass;
      const uint2 *meta = reinterpret_cast<const uint2 *>(buf);
      const double2 *terms = reinterpret_cast<const double2 *>(buf + 256 * np);
      int q = 0;
      while (q < np) {
        const uint2 m0 = meta[q * 32 + lane];
        const int w0 = (int)((m0.x >> 16) & 0x7FFFu);
        const double2 *t0 = terms + m0.y;
        if (!(m0.x >> 31) && q + 1 < np) {
          const uint2 m1 = meta[(q + 1) * 32 + lane];
          const int w1 = (int)((m1.x >> 16) & 0x7FFFu);
          const double2 *t1 = terms + m1.y;
          typename R::Acc a0, a1;
          r.init(a0);
          r.init(a1);
          int t = 0;
#pragma unroll 2
          for (; t < w1; ++t) {
            r.term(a0, t0[32 * t], lvl);
            r.term(a1, t1[32 * t], lvl);
          }
#pragma unroll 2
          for (; t < w0; ++t) r.term(a0, t0[32 * t], lvl);
          if ((m0.x & 0xFFFFu) != 0xFFFFu) r.store(m0.x & 0xFFFFu, a0);
          if ((m1.x & 0xFFFFu) != 0xFFFFu) r.store(m1.x & 0xFFFFu, a1);
          q += 2;
          if (m1.x >> 31) {
            __syncwarp();
            ++lvl;
          }
        } else {
          typename R::Acc a0;
          r.init(a0);
#pragma unroll 4
          for (int t = 0; t < w0; ++t) r.term(a0, t0[32 * t], lvl);
          if ((m0.x & 0xFFFFu) != 0xFFFFu) r.store(m0.x & 0xFFFFu, a0);
          q += 1;
          if (m0.x >> 31) {
            __syncwarp();
            ++lvl;
          }
        }
      }
    }
    ++pp.gc;
  }
  __syncwarp();
}

__device__ __forceinline__ int term_src(const double2 &tv) { return (int)__double_as_longlong(tv.y); }

template <int F, int K>
__device__ __forceinline__ void tangentialK(const double *s, int N, int a, double (&a1)[K], double (&a2)[K]) {
  if constexpr (F == 0) {
    double y0[K];
    ldk<K>(s + a * K, y0);
    ldk<K>(s + (N + a) * K, a1);
    ldk<K>(s + (2 * N + a) * K, a2);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      a1[k] -= y0[k];
      a2[k] -= y0[k];
    }
  } else if constexpr (F == 1) {
    ldk<K>(s + (N + a) * K, a1);
    ldk<K>(s + (2 * N + a) * K, a2);
  } else if constexpr (F == 2) {
    ldk<K>(s + a * K, a1);
    ldk<K>(s + (2 * N + a) * K, a2);
  } else {
    ldk<K>(s + a * K, a1);
    ldk<K>(s + (N + a) * K, a2);
  }
}

template <int P, int K>
__device__ __forceinline__ void load_async(const double *__restrict__ Fd, int64_t e0, int nk, int64_t cs, double *s,
                                           int lane) {
  using D = DS<P>;
  constexpr int N = D::N, LD = D::LD;
  for (int c = 0; c < 3; ++c) {
    const double *src = Fd + c * cs + e0 * LD;
    for (int i = lane; i < nk * LD; i += 32) {
      const int k = i / LD, b = i - k * LD;
      if (b < N) cp_async8(s + (c * N + b) * K + k, src + i);
    }
  }
}

// ---- row functors ---------------------------------------------------------
template <int K>
struct CurlRow {   // scalar slots of the warp workspace
  double *ws;
  struct Acc {
    double v[K];
  };
  __device__ __forceinline__ void init(Acc &a) const {
#pragma unroll
    for (int k = 0; k < K; ++k) a.v[k] = 0.0;
  }
  __device__ __forceinline__ void term(Acc &a, const double2 tv, int) const {
    double x[K];
    ldk<K>(ws + term_src(tv) * K, x);
#pragma unroll
    for (int k = 0; k < K; ++k) a.v[k] = fma(tv.x, x[k], a.v[k]);
  }
  __device__ __forceinline__ void store(unsigned d, const Acc &a) const { stk<K>(ws + d * K, a.v); }
};

template <int F, int K>
struct TraceRow {   // stage 0: tangential components of the volume slots; later: pair scratch
  const double *ws;
  double2 *scr2;
  int N;
  struct Acc {
    double t1[K], t2[K];
  };
  __device__ __forceinline__ void init(Acc &a) const {
#pragma unroll
    for (int k = 0; k < K; ++k) a.t1[k] = a.t2[k] = 0.0;
  }
  __device__ __forceinline__ void term(Acc &a, const double2 tv, int lvl) const {
    const int sr = term_src(tv);
    if (lvl == 0) {
      double a1[K], a2[K];
      tangentialK<F, K>(ws, N, sr, a1, a2);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        a.t1[k] = fma(tv.x, a1[k], a.t1[k]);
        a.t2[k] = fma(tv.x, a2[k], a.t2[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double2 v = scr2[sr * K + k];
        a.t1[k] = fma(tv.x, v.x, a.t1[k]);
        a.t2[k] = fma(tv.x, v.y, a.t2[k]);
      }
    }
  }
  __device__ __forceinline__ void store(unsigned d, const Acc &a) const {
#pragma unroll
    for (int k = 0; k < K; ++k) scr2[d * K + k] = make_double2(a.t1[k], a.t2[k]);
  }
};

template <int K>
struct LiftRow {   // stage 0: (A, B) pairs; later: pair scratch
  const double2 *AB2;
  double2 *scr2;
  struct Acc {
    double la[K], lb[K];
  };
  __device__ __forceinline__ void init(Acc &a) const {
#pragma unroll
    for (int k = 0; k < K; ++k) a.la[k] = a.lb[k] = 0.0;
  }
  __device__ __forceinline__ void term(Acc &a, const double2 tv, int lvl) const {
    const double2 *in = lvl == 0 ? AB2 : scr2;
    const int sr = term_src(tv);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double2 v = in[sr * K + k];
      a.la[k] = fma(tv.x, v.x, a.la[k]);
      a.lb[k] = fma(tv.x, v.y, a.lb[k]);
    }
  }
  __device__ __forceinline__ void store(unsigned d, const Acc &a) const {
#pragma unroll
    for (int k = 0; k < K; ++k) scr2[d * K + k] = make_double2(a.la[k], a.lb[k]);
  }
};

// staged trace of face F (program 5+F) for the warp's elements -> trace buffer
template <int P, int F, int K>
__device__ __forceinline__ void warp_strace(const DevStream &S, const DevSProg &sp, bool more, bool active, Pipe &pp,
                                            int tid, int lane, double *ws, double *tr, int64_t e0, int nk) {
  using D = DS<P>;
  constexpr int N = D::N, NF = D::NF;
  double2 *scr2 = reinterpret_cast<double2 *>(ws + D::SCR * K);
  run_prog(S, 5 + F, more, active, pp, tid, lane, TraceRow<F, K>{ws, scr2, N});
  if (active)
    for (int i = lane; i < nk * NF; i += 32) {
      const int k = i / NF, g = i - k * NF;
      const double2 v = scr2[__ldg(sp.out + g) * K + k];
      double *o = tr + ((e0 + k) * 4 + F) * 2 * NF;
      o[g] = v.x;
      o[NF + g] = v.y;
    }
  __syncwarp();
}

// staged lift of face F (program 1+F) of the pairs (A, B) into the accumulator
template <int P, int F, int K>
__device__ __forceinline__ void warp_slift(const DevStream &S, const DevSProg &sp, bool more, bool active, Pipe &pp,
                                           int tid, int lane, double *ws) {
  using D = DS<P>;
  constexpr int N = D::N;
  double2 *scr2 = reinterpret_cast<double2 *>(ws + D::SCR * K);
  const double2 *AB2 = reinterpret_cast<const double2 *>(ws + D::SAB * K);
  run_prog(S, 1 + F, more, active, pp, tid, lane, LiftRow<K>{AB2, scr2});
  if (active) {
    const double a0 = sT1[F][0], a1 = sT1[F][1], a2 = sT1[F][2];
    const double b0 = sT2[F][0], b1 = sT2[F][1], b2 = sT2[F][2];
    double *acc = ws + D::ACC * K;
    for (int i = lane; i < N * K; i += 32) {
      const int b = i / K, k = i - b * K;
      const int sl = __ldg(sp.out + b);
      if (sl == 0xFFFF) continue;
      const double2 v = scr2[sl * K + k];
      if (a0 != 0.0 || b0 != 0.0) acc[b * K + k] += a0 * v.x + b0 * v.y;
      if (a1 != 0.0 || b1 != 0.0) acc[(N + b) * K + k] += a1 * v.x + b1 * v.y;
      if (a2 != 0.0 || b2 != 0.0) acc[(2 * N + b) * K + k] += a2 * v.x + b2 * v.y;
    }
  }
  __syncwarp();
}

// face fields (A, B) of face f for the warp's elements -> pairs at ws[SAB]
template <int P, bool UP, int K>
__device__ __forceinline__ void warp_flux(const StageArgs &a, const double *__restrict__ trY, const double *sG,
                                          double *ws, int64_t e0, int nk, int f, int lane) {
  using D = DS<P>;
  constexpr int NF = D::NF;
  const bool stageE = a.stage == STAGE_E;
  const double mirrorY = stageE ? 1.0 : -1.0, mirrorX = stageE ? -1.0 : 1.0;
  const double sf = (f & 1) ? -1.0 : 1.0;
  double2 *sAB = reinterpret_cast<double2 *>(ws + D::SAB * K);
  for (int i = lane; i < K * NF; i += 32) {
    const int k = i / NF, gm = i - k * NF;
    double A = 0.0, B = 0.0;
    if (k < nk) {
      const int64_t e = e0 + k;
      const int nb = a.nbr[4 * e + f];
      const int gf = a.nbrf[4 * e + f];
      double w = 0.5, kk = 0.0;
      const double *gk = sG + k * D::GEO;
      if (UP) {
        const double Zm = gk[9], Zp = nb >= 0 ? a.geo[nb].Z : Zm;
        if (stageE) {
          w = Zp / (Zm + Zp);
          kk = 1.0 / (Zm + Zp);
        } else {
          const double Ym = 1.0 / Zm, Yp = 1.0 / Zp;
          w = Yp / (Ym + Yp);
          kk = 1.0 / (Ym + Yp);
        }
      }
      const double *to = trY + (e * 4 + f) * 2 * NF;
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
        const double *hf = a.HF + (int64_t)a.fid[4 * e + f] * 2 * NF;
        h1 = __ldg(hf + gm);
        h2 = __ldg(hf + NF + gm);
      }
      A = -sf * (w * (n2 - o2) - h2);
      B = sf * (w * (n1 - o1) - h1);
      if (UP) {
        const double *xo = a.trX + (e * 4 + f) * 2 * NF;
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
        const double ps = (stageE ? 1.0 : -1.0) * (gk[6] > 0 ? 1.0 : -1.0);
        A += ps * (j1 * M[0] + j2 * M[1]);
        B += ps * (j1 * M[1] + j2 * M[2]);
      }
    }
    sAB[gm * K + k] = make_double2(A, B);
  }
  __syncwarp();
}

template <int P>
__host__ __device__ constexpr size_t warp_doubles(int K) {
  return (size_t)K * (DS<P>::WS + DS<P>::GEO);
}

template <int P, bool UP, int K>
__global__ void __launch_bounds__(512, 1) stream_kernel(StageArgs a, DevProgs pr, DevStream S,
                                                        const double *__restrict__ trY, double *__restrict__ trOut,
                                                        int chunk_bytes) {
  using D = DS<P>;
  constexpr int N = D::N, LD = D::LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  Pipe pp;
  pp.chunk_bytes = chunk_bytes;
  pp.gc = 0;
  double *ws = reinterpret_cast<double *>(smem_raw + 128 + 2 * (size_t)chunk_bytes) + warp * warp_doubles<P>(K);
  double *sG = ws + (size_t)K * D::WS;
  double *sACC = ws + D::ACC * K;
  const int64_t cs = a.n_tet * LD;
  const bool stageE = a.stage == STAGE_E;
  const bool upd = a.out_mode == OUT_UPDATE;
  const int64_t per = (int64_t)nw * K;
  const int64_t nbatch = (a.n_tet + per - 1) / per;
  if (tid == 0) {
    mbar_init(pipe_mbar(0), 1);
    mbar_init(pipe_mbar(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < nbatch) {
    const StreamChunk c = S.chunks[0];
    tma_load(pipe_buf(pp, 0), S.base + c.off, c.bytes, pipe_mbar(0));
  }
  for (int64_t bt = blockIdx.x; bt < nbatch; bt += gridDim.x) {
    const bool more = bt + gridDim.x < nbatch;
    const int64_t e0 = (bt * nw + warp) * K;
    const int nk = e0 < a.n_tet ? (int)((a.n_tet - e0) < K ? (a.n_tet - e0) : K) : 0;
    const bool active = nk > 0;
    if (active) {
      load_async<P, K>(a.Y, e0, nk, cs, ws, lane);
      for (int i = lane; i < nk * D::GEO; i += 32) {
        const int k = i / D::GEO, j = i - k * D::GEO;
        sG[i] = reinterpret_cast<const double *>(a.geo + e0 + k)[j];
      }
      cp_async_wait_all();
    }
    __syncwarp();
    // S1: reference curl by the recurrence sweeps (program 0)
    run_prog(S, 0, more, active && a.do_curl, pp, tid, lane, CurlRow<K>{ws});
    if (active && !a.do_curl) {
      for (int i = lane; i < 3 * N * K; i += 32) sACC[i] = 0.0;
      __syncwarp();
    }
    // Ŷ is dead (traces come from the buffer): stage X in its slots while the fluxes run
    if (active && upd) load_async<P, K>(a.X, e0, nk, cs, ws, lane);
    // S3-S5: flux and lift per face (programs 1..4)
    const bool fl = active && a.do_flux;
    if (fl) warp_flux<P, UP, K>(a, trY, sG, ws, e0, nk, 0, lane);
    warp_slift<P, 0, K>(S, pr.slift[0], more, fl, pp, tid, lane, ws);
    if (fl) warp_flux<P, UP, K>(a, trY, sG, ws, e0, nk, 1, lane);
    warp_slift<P, 1, K>(S, pr.slift[1], more, fl, pp, tid, lane, ws);
    if (fl) warp_flux<P, UP, K>(a, trY, sG, ws, e0, nk, 2, lane);
    warp_slift<P, 2, K>(S, pr.slift[2], more, fl, pp, tid, lane, ws);
    if (fl) warp_flux<P, UP, K>(a, trY, sG, ws, e0, nk, 3, lane);
    warp_slift<P, 3, K>(S, pr.slift[3], more, fl, pp, tid, lane, ws);
    // S2 + S6: inverse mass with geometry, then update or write
    if (active) {
      if (upd) cp_async_wait_all();
      __syncwarp();
      for (int i = lane; i < nk * N; i += 32) {
        const int k = i / N, b = i - k * N;
        const double *gk = sG + k * D::GEO;
        const double cm = stageE ? gk[7] : -gk[8];
        const double v0 = sACC[b * K + k], v1 = sACC[(N + b) * K + k], v2 = sACC[(2 * N + b) * K + k];
        const double x0 = cm * (gk[0] * v0 + gk[1] * v1 + gk[2] * v2);
        const double x1 = cm * (gk[1] * v0 + gk[3] * v1 + gk[4] * v2);
        const double x2 = cm * (gk[2] * v0 + gk[4] * v1 + gk[5] * v2);
        const int64_t o = (e0 + k) * LD + b;
        if (upd) {
          double *y = ws + b * K + k;
          const double y0 = y[0] + a.dt * x0, y1 = y[N * K] + a.dt * x1, y2 = y[2 * N * K] + a.dt * x2;
          y[0] = y0;
          y[N * K] = y1;
          y[2 * N * K] = y2;
          a.X[o] = y0;
          a.X[cs + o] = y1;
          a.X[2 * cs + o] = y2;
        } else if (a.out_mode == OUT_WRITE) {
          a.dX[o] = x0;
          a.dX[cs + o] = x1;
          a.dX[2 * cs + o] = x2;
        } else {
          a.dX[o] += x0;
          a.dX[cs + o] += x1;
          a.dX[2 * cs + o] += x2;
        }
      }
    }
    __syncwarp();
    // traces of the updated field for the next stage (programs 5..8)
    const bool tw = active && upd && trOut;
    warp_strace<P, 0, K>(S, pr.strace[0], more, tw, pp, tid, lane, ws, trOut, e0, nk);
    warp_strace<P, 1, K>(S, pr.strace[1], more, tw, pp, tid, lane, ws, trOut, e0, nk);
    warp_strace<P, 2, K>(S, pr.strace[2], more, tw, pp, tid, lane, ws, trOut, e0, nk);
    warp_strace<P, 3, K>(S, pr.strace[3], more, tw, pp, tid, lane, ws, trOut, e0, nk);
  }
}

// entry traces of a field (programs 5..8 only; the other chunks are skipped by
// issuing the trace chunks directly: this kernel uses its own schedule offset)
template <int P, int K>
__global__ void __launch_bounds__(512, 1) stream_trace_kernel(const double *__restrict__ X, double *tr, int64_t n_tet,
                                                              DevProgs pr, DevStream S, int chunk_bytes) {
  using D = DS<P>;
  constexpr int LD = D::LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // restrict the schedule to programs 5..8 by shifting the chunk table
  DevStream T = S;
  const int c5 = S.first[5];
  T.chunks = S.chunks + c5;
  T.nchunk = S.nchunk - c5;
  for (int i = 0; i < 9; ++i) T.first[i] = S.first[i] - c5;
  Pipe pp;
  pp.chunk_bytes = chunk_bytes;
  pp.gc = 0;
  double *ws = reinterpret_cast<double *>(smem_raw + 128 + 2 * (size_t)chunk_bytes) + warp * warp_doubles<P>(K);
  const int64_t cs = n_tet * LD;
  const int64_t per = (int64_t)nw * K;
  const int64_t nbatch = (n_tet + per - 1) / per;
  if (tid == 0) {
    mbar_init(pipe_mbar(0), 1);
    mbar_init(pipe_mbar(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < nbatch) tma_load(pipe_buf(pp, 0), T.base + T.chunks[0].off, T.chunks[0].bytes, pipe_mbar(0));
  for (int64_t bt = blockIdx.x; bt < nbatch; bt += gridDim.x) {
    const bool more = bt + gridDim.x < nbatch;
    const int64_t e0 = (bt * nw + warp) * K;
    const int nk = e0 < n_tet ? (int)((n_tet - e0) < K ? (n_tet - e0) : K) : 0;
    if (nk > 0) {
      load_async<P, K>(X, e0, nk, cs, ws, lane);
      cp_async_wait_all();
    }
    __syncwarp();
    warp_strace<P, 0, K>(T, pr.strace[0], more, nk > 0, pp, tid, lane, ws, tr, e0, nk);
    warp_strace<P, 1, K>(T, pr.strace[1], more, nk > 0, pp, tid, lane, ws, tr, e0, nk);
    warp_strace<P, 2, K>(T, pr.strace[2], more, nk > 0, pp, tid, lane, ws, tr, e0, nk);
    warp_strace<P, 3, K>(T, pr.strace[3], more, nk > 0, pp, tid, lane, ws, tr, e0, nk);
  }
}

int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// warps per CTA: as many element workspaces as fit next to the two chunk buffers
template <int P, int K>
int pick_nw(dgm_ctx *c, size_t &smem) {
  const size_t fixed = 128 + 2 * (size_t)c->stream.max_bytes;
  const size_t per = sizeof(double) * warp_doubles<P>(K);
  int nw = env_int("DGM_ST_NW", 0);
  const size_t cap = 227 * 1024;
  if (nw <= 0) nw = fixed + per <= cap ? (int)((cap - fixed) / per) : 0;
  if (nw > 16) nw = 16;
  smem = fixed + per * (size_t)nw;
  return (nw >= 1 && smem <= cap) ? nw : 0;
}

template <int P, int K>
dgm_status stream_go(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st) {
  size_t smem = 0;
  const int nw = pick_nw<P, K>(c, smem);
  if (nw < 1) return set_err(c, DGM_EINVAL, "stream kernel: workspace does not fit in shared memory");
  const int64_t nb = (c->n_tet + (int64_t)nw * K - 1) / ((int64_t)nw * K);
  const unsigned grid = (unsigned)(nb < c->sms ? nb : c->sms);
  if (a.upwind) {
    auto kern = stream_kernel<P, true, K>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * nw, smem, st>>>(a, c->progs, c->stream, trY, trOut, c->stream.max_bytes);
  } else {
    auto kern = stream_kernel<P, false, K>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 32 * nw, smem, st>>>(a, c->progs, c->stream, trY, trOut, c->stream.max_bytes);
  }
  c->launches++;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("stream_kernel: ") + cudaGetErrorString(e));
}

template <int P, int K>
dgm_status stream_tr_go(dgm_ctx *c, const double *X, double *tr, cudaStream_t st) {
  size_t smem = 0;
  const int nw = pick_nw<P, K>(c, smem);
  if (nw < 1) return set_err(c, DGM_EINVAL, "stream kernel: workspace does not fit in shared memory");
  const int64_t nb = (c->n_tet + (int64_t)nw * K - 1) / ((int64_t)nw * K);
  const unsigned grid = (unsigned)(nb < c->sms ? nb : c->sms);
  auto kern = stream_trace_kernel<P, K>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<grid, 32 * nw, smem, st>>>(X, tr, c->n_tet, c->progs, c->stream, c->stream.max_bytes);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("stream_trace_kernel: ") + cudaGetErrorString(e));
}

template <int P>
dgm_status stream_stage_p(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st) {
  switch (env_int("DGM_ST_KW", 1)) {
    case 2: return stream_go<P, 2>(c, a, trY, trOut, st);
    default: return stream_go<P, 1>(c, a, trY, trOut, st);
  }
}

template <int P>
dgm_status stream_traces_p(dgm_ctx *c, const double *X, double *tr, cudaStream_t st) {
  switch (env_int("DGM_ST_KW", 1)) {
    case 2: return stream_tr_go<P, 2>(c, X, tr, st);
    default: return stream_tr_go<P, 1>(c, X, tr, st);
  }
}

}  // namespace

dgm_status launch_stream_stage(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st) {
  switch (c->p) {
    case 7: return stream_stage_p<7>(c, a, trY, trOut, st);
    case 8: return stream_stage_p<8>(c, a, trY, trOut, st);
    case 9: return stream_stage_p<9>(c, a, trY, trOut, st);
    case 10: return stream_stage_p<10>(c, a, trY, trOut, st);
    default: return DGM_EORDER;
  }
}

dgm_status launch_stream_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st) {
  switch (c->p) {
    case 7: return stream_traces_p<7>(c, X, tr, st);
    case 8: return stream_traces_p<8>(c, X, tr, st);
    case 9: return stream_traces_p<9>(c, X, tr, st);
    case 10: return stream_traces_p<10>(c, X, tr, st);
    default: return DGM_EORDER;
  }
}

}  // namespace dgm
