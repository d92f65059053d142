// Streamed lane-per-element curl sweeps (high orders), sm_100a FP64.
//
// The reference curl ĉ = curl̂ Ŷ by the paper's recurrences, one
// directional sweep per warp, lane = element (32 elements per warp, every lane the
// same generated straight-line code with warp-uniform immediate coefficients; the
// SIMT form of the paper's template-metaprogrammed loops).  See
// gen/sweepgen.py for why a sweep is a streaming computation: it consumes its input
// component and produces its outputs in reverse memory order, with about two degree
// levels of intermediate values live in registers.
//
// Input: Ŷ in the ABI layout [3][n_tet][LD].  Output: ĉ [3][n_tet][LDC] (N' = N(p-1)
// real modes, zero padding to LDC), in the accumulator frame of the stage GEMM (before
// G' and ±1/m).  A warp pair computes one output component m of 32 elements:
//     m = 0: ĉx = ∂y Ŷz - ∂z Ŷy,  m = 1: ĉy = ∂z Ŷx - ∂x Ŷz,  m = 2: ĉz = ∂x Ŷy - ∂y Ŷx
// warp 0 of the pair runs the + sweep, warp 1 the - sweep.  Each warp streams its input
// component through a 3-slot ring of 16-mode chunks in shared memory and writes its
// outputs into a 2-slot ring; per output chunk the two warps meet at a named barrier
// and each flushes half the chunk as ĉ = w₊ - w₋ (written once, coalesced).  A CTA
// holds NPAIR pairs working on the same m (4 groups of 32 elements), so its 8 warps
// run two instruction streams in near lockstep.
//
// Measured at p = 10, C5 (tools/curlbench, ms per launch; earlier session): coefficients
// through the constant bank with the warps spread over all directions 19.4; the same
// with the CTA's pairs on one m 7.5; a shared-memory coefficient table 8.8; immediates
// 5.8.  Splitting ĉ by sign so that every warp of a CTA runs the same direction without
// barriers (two output buffers, twice the output writes) 8.4.  Round 2, same binary
// harness on one box (profiles/r02_curl_variants.txt): immediates 8.06, the constant
// table in order of first use (gen/sweepgen.py Consts, the default) 6.73; a CTA-wide
// lockstep barrier instead of the pair barrier changes neither.  The sweeps sit at
// 8-10% of the FP64 pipe: 255 registers (a two-degree-level window of u per lane) leave
// two warps per scheduler, and every instruction-line fetch or constant load is exposed.
// Warp pairs per CTA (DGM_CURL_NPAIR, same 8 warps per SM): 4 pairs 6.71 ms, 2 pairs
// 9.90, 1 pair 18.5 — CTAs on one SM then run different output components, i.e. more
// distinct instruction streams and constant tables per SM.
#pragma once
#include <cstdint>
#include <string>

#include "dgm_internal.h"

namespace dgm {
namespace curl {

constexpr int CH = 16;            // modes per chunk
constexpr int CS = 33;            // padded element stride of an output slot ([mode][element])
constexpr int SLOT = CH * CS;     // doubles per output slot
constexpr int RS = 18;            // input slot row stride (16 modes + pad, 16-byte aligned rows)
constexpr int SLOT_IN = 32 * RS;  // doubles per input slot ([element][RS])
constexpr int RIN = 3, ROUT = 2;  // ring slots
#ifndef DGM_CURL_NPAIR
#define DGM_CURL_NPAIR 4
#endif
constexpr int NPAIR = DGM_CURL_NPAIR;   // warp pairs per CTA
constexpr int WARP_SMEM = RIN * SLOT_IN + ROUT * SLOT;   // doubles of ring per warp

// a 64-bit immediate operand (the sweeps' coefficients): volatile so ptxas keeps it an
// immediate (two uniform moves) instead of pooling it in the constant bank
template <unsigned long long B>
__device__ __forceinline__ double kimm() {
  double x;
  asm volatile("mov.b64 %0, %1;" : "=d"(x) : "n"(B));
  return x;
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NW>
__device__ __forceinline__ void wait_groups() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NW) : "memory");
}
// named barrier of warp pair q (ids 1..NPAIR; 0 is __syncthreads)
#ifdef CURL_CTA_SYNC   // experiments: all pairs of the CTA in lockstep (one named barrier of the CTA)
__device__ __forceinline__ void pair_barrier(int) { asm volatile("bar.sync 1, %0;\n" ::"n"(64 * NPAIR) : "memory"); }
#else
__device__ __forceinline__ void pair_barrier(int q) { asm volatile("bar.sync %0, 64;\n" ::"r"(q + 1) : "memory"); }
#endif

template <int P>
struct Dims {
  static constexpr int N = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int LD = (N + 3) & ~3;
  static constexpr int NPR = P * (P + 1) * (P + 2) / 6;
  static constexpr int LDC = (NPR + CH - 1) / CH * CH;
};

// The generated sweep's view of the streams: every offset is a compile-time constant;
// shared memory goes through 32-bit addresses and ld/st.shared.
// Input chunk Q of a warp = modes [16Q, 16Q+16) of its 32 elements (32 rows of 128 B):
// 16-byte cp.async, 8 per lane (lane l copies piece l%8 of rows l/8 + 4i), into slot
// Q % RIN laid out [element][RS]; a lane then reads its own row (2-way bank conflicts
// at RS = 18).  Measured alternatives: 8-byte copies into a conflict-free transposed
// layout (16 copies + address arithmetic per lane and chunk), and one bulk copy per
// row (the compiler serialises per-lane bulk copies through the uniform datapath).
template <int P>
struct IO {
  using D = Dims<P>;
  const double *src;   // Ŷ_c + (e0 + lane/8) LD + 2 (lane%8): this lane's copy source
  double *dst;         // ĉ_m + (e0 + lane/8) LDC + 8w + lane%8: this lane's flush target
  unsigned rin_w;      // input ring + (lane/8) RS + 2 (lane%8)  (copy destination, slot 0)
  unsigned rin;        // input ring + lane RS                   (this lane's row, slot 0)
  unsigned rout_w;     // own output ring + lane
  unsigned ra, rb;     // output rings of warp 0 (+) / warp 1 (-) + (8w + lane%8) CS + lane/8
  int nel;             // valid elements of the group (1..32)
  int pair;            // warp pair within the CTA (named barrier)
  int l8, l7;          // lane/8, lane%8

  template <int Q>
  __device__ __forceinline__ void issue() const {
    const unsigned d = rin_w + 8u * (unsigned)((Q % RIN) * SLOT_IN);
    const double *s = src + CH * Q;
    const bool mode_ok = CH * Q + 15 < D::LD || CH * Q + 2 * l7 < D::LD;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int bytes = mode_ok && 4 * i + l8 < nel ? 16 : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d + 8u * (unsigned)(4 * i * RS)),
                   "l"(s + 4 * i * D::LD), "r"(bytes)
                   : "memory");
    }
  }
  template <int K>
  __device__ __forceinline__ void prime() const {
    issue<K>();
    commit();
    if constexpr (K >= 1) issue<K - 1>();
    commit();
  }
  // first use of chunk K: it has landed (chunk K-1 may still be in flight); the slot of
  // chunk K+1 (never read again) takes chunk K-2.  The returned token is the read base,
  // passed through a volatile asm: the chunk's reads depend on it, so they cannot move
  // above the wait, but may be hoisted freely between this switch and their use.
  template <int K>
  __device__ __forceinline__ unsigned sw() const {
    wait_groups<1>();
    __syncwarp();
    if constexpr (K >= 2) issue<K - 2>();
    commit();
    unsigned t;
    asm volatile("mov.b32 %0, %1;\n" : "=r"(t) : "r"(rin) : "memory");
    return t;
  }
  template <int G>
  __device__ __forceinline__ double v(unsigned tok) const {
    double x;
    asm("ld.shared.f64 %0, [%1+%2];\n" : "=d"(x) : "r"(tok), "n"(8 * (((G / CH) % RIN) * SLOT_IN + (G % CH))));
    return x;
  }
  template <int B>
  __device__ __forceinline__ void o(double x) const {
    asm volatile("st.shared.f64 [%0+%1], %2;\n" ::"r"(rout_w), "n"(8 * (((B / CH) % ROUT) * SLOT + (B % CH) * CS)),
                 "d"(x));
  }
  // output chunk J complete in both warps of the pair: warp w writes modes 8w..8w+7 of
  // it for the 32 elements (8 consecutive modes of 4 elements per instruction)
  template <int J>
  __device__ __forceinline__ void flush() const {
    pair_barrier(pair);
    double *d = dst + CH * J;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double a, b;
      const unsigned off = 8u * (unsigned)((J % ROUT) * SLOT + 4 * i);
      asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a) : "r"(ra + off));
      asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(b) : "r"(rb + off));
      if (4 * i + l8 < nel) d[4 * i * D::LDC] = a - b;
    }
  }
  __device__ __forceinline__ void drain() const {
    wait_groups<0>();
    __syncwarp();
  }
};

}  // namespace curl
}  // namespace dgm

// Kernel and launcher for order P, given the generated csweep_p{P}_d{0,1,2}.
// Dynamic shared memory: per warp its rings.
#define DGM_CURL_INSTANTIATE(P)                                                                              \
  namespace dgm {                                                                                            \
  namespace curl {                                                                                           \
  constexpr size_t kSmem##P = sizeof(double) * (size_t)(2 * NPAIR * WARP_SMEM);                              \
  __global__ void __launch_bounds__(64 * NPAIR, 1) curl_kernel_p##P(const double *__restrict__ Y,            \
                                                                 double *__restrict__ C, int64_t n_tet) {  \
    using D = Dims<P>;                                                                                       \
    extern __shared__ __align__(16) double sm[];                                                             \
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, q = wid >> 1, w = wid & 1;                    \
    const int64_t groups = (n_tet + 31) / 32, batches = (groups + NPAIR - 1) / NPAIR;                        \
    const int64_t cs = n_tet * D::LD, ccs = n_tet * D::LDC;                                                  \
    const unsigned sin = (unsigned)__cvta_generic_to_shared(sm + wid * WARP_SMEM);                           \
    const unsigned so0 = (unsigned)__cvta_generic_to_shared(sm + (2 * q) * WARP_SMEM + RIN * SLOT_IN);       \
    const unsigned so1 = (unsigned)__cvta_generic_to_shared(sm + (2 * q + 1) * WARP_SMEM + RIN * SLOT_IN);   \
    for (int64_t it = blockIdx.x; it < 3 * batches; it += gridDim.x) {                                       \
      const int m = (int)(it % 3);                                                                           \
      const int64_t e0 = ((it / 3) * NPAIR + q) * 32;                                                        \
      if (e0 < n_tet) {                                                                                      \
        /* m = 0: +∂y Ŷz, -∂z Ŷy;  m = 1: +∂z Ŷx, -∂x Ŷz;  m = 2: +∂x Ŷy, -∂y Ŷx */                          \
        const int d = w == 0 ? (m + 1) % 3 : (m + 2) % 3;                                                    \
        const int c = w == 0 ? (m + 2) % 3 : (m + 1) % 3;                                                    \
        IO<P> io;                                                                                            \
        io.l8 = lane >> 3;                                                                                   \
        io.l7 = lane & 7;                                                                                    \
        io.pair = q;                                                                                         \
        io.nel = (int)(n_tet - e0 < 32 ? n_tet - e0 : 32);                                                   \
        io.src = Y + c * cs + (e0 + (lane >> 3)) * D::LD + 2 * (lane & 7);                                   \
        io.dst = C + m * ccs + (e0 + (lane >> 3)) * D::LDC + 8 * w + (lane & 7);                             \
        io.rin_w = sin + 8u * (unsigned)((lane >> 3) * RS + 2 * (lane & 7));                                 \
        io.rin = sin + 8u * (unsigned)(lane * RS);                                                           \
        io.rout_w = (w ? so1 : so0) + 8u * (unsigned)lane;                                                   \
        const unsigned fo = 8u * (unsigned)((8 * w + (lane & 7)) * CS + (lane >> 3));                        \
        io.ra = so0 + fo;                                                                                    \
        io.rb = so1 + fo;                                                                                    \
        if (d == 0) csweep_p##P##_d0(io);                                                                    \
        else if (d == 1) csweep_p##P##_d1(io);                                                               \
        else csweep_p##P##_d2(io);                                                                           \
      }                                                                                                      \
      __syncthreads(); /* all pairs done with their rings; the next item starts in step */                   \
    }                                                                                                        \
  }                                                                                                          \
  }                                                                                                          \
  dgm_status launch_curl_p##P(dgm_ctx *c, const double *Y, double *C, cudaStream_t st) {                     \
    static int occ = 0;                                                                                      \
    if (!occ) {                                                                                              \
      cudaFuncSetAttribute(curl::curl_kernel_p##P, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                           (int)curl::kSmem##P);                                                             \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, curl::curl_kernel_p##P, 64 * curl::NPAIR,          \
                                                    curl::kSmem##P);                                         \
      if (occ < 1) occ = 1;                                                                                  \
    }                                                                                                        \
    const int64_t items = 3 * (((c->n_tet + 31) / 32 + curl::NPAIR - 1) / curl::NPAIR);                      \
    int64_t grid = (int64_t)c->sms * occ;                                                                    \
    if (grid > items) grid = items;                                                                          \
    if (grid < 1) return DGM_OK;                                                                             \
    curl::curl_kernel_p##P<<<(unsigned)grid, 64 * curl::NPAIR, curl::kSmem##P, st>>>(Y, C, c->n_tet);        \
    c->launches++;                                                                                           \
    cudaError_t e = cudaGetLastError();                                                                      \
    return e == cudaSuccess ? DGM_OK                                                                         \
                            : set_err(c, DGM_ECUDA, std::string("curl_kernel: ") + cudaGetErrorString(e));  \
  }                                                                                                          \
  }
