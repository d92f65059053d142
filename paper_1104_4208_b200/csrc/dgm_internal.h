// Internal declarations shared by the host setup (dgm_host.cpp) and the
// kernels (dgm_kernels.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/dgm.h"

namespace dgm {

// One level-scheduled ELL program (see gen/plan.py): pass ps covers rows
// [ps*32, ps*32+32); its terms are stored [term][lane] from off[ps]*32.
struct HostProg {
  int npass, nterm;
  const uint16_t *dst, *cnt, *src;
  const double *coef;
  const int32_t *off;
  const uint8_t *sync;
};
// staged (sum-factorised) program: stage 0 reads the n_in inputs, later stages and
// all destinations live in an n_scr-slot scratch; out[i] = scratch slot of output i
struct HostSProg {
  HostProg prog;
  int n_in, n_scr;
  const uint16_t *out;
};
struct HostProgSet {
  int p, acc;
  HostProg curl;
  HostProg trace[4];
  HostProg lift[4];
  HostSProg strace[4];
  HostSProg slift[4];
  const double *norms;
};

struct DevProg {
  int npass;
  const uint16_t *__restrict__ dst;
  const uint16_t *__restrict__ cnt;
  const uint16_t *__restrict__ src;
  const double *__restrict__ coef;
  const int32_t *__restrict__ off;
  const uint8_t *__restrict__ sync;
  // the same terms packed as 16-byte {coef, src} pairs: one 128-bit load per term
  const double2 *__restrict__ term;
  // per row {dst | cnt << 16, first term index (off*32 + lane)}: one 64-bit load per row
  const uint2 *__restrict__ meta;
  // per DAG level {first pass, last pass}
  const int2 *__restrict__ lvl;
  int nlev;
};
struct DevSProg {
  DevProg prog;
  int n_in, n_scr;
  const uint16_t *__restrict__ out;
};
// Table stream for the high-order streamed kernels (dgm_stream.cu): the programs
// curl, slift[0..3], strace[0..3] cut into chunks of whole passes; each chunk is
// [meta: npass*32 uint2 {dst | cnt<<16 | level_end<<31, first term (chunk-relative)}]
// [terms: double2 {coef, src}], copied into shared memory by one bulk TMA copy.
struct StreamChunk {
  uint32_t off, bytes;
  int32_t npass, pad;
};
struct DevStream {
  const char *__restrict__ base;
  const StreamChunk *__restrict__ chunks;
  int first[9], count[9];
  int nchunk, max_bytes;
};

// Dense-contraction engine (dgm_dense.cu): per-context operator matrices assembled
// from the exact programs.  Rows are component-blocked and padded to the k-tile
// (Nk = N, NFk = NF rounded up to 16).  B1 [3Nk+8NFk][3Np]: rows c*Nk+β (curl input),
// k1a + j*NFk + γ (face field j = f*2+{A,B}); columns m*Np+β (Np = N rounded up to
// 32 stage_nh).  B2 [3Nk][nc2]: rows c*Nk+β, columns (f*2+k)*NF+γ (trace-buffer order).
// ktl/ktoff: per n-tile the non-zero k-tiles with a 12-bit mask per warp column of non-zero 16x8
// column groups (sel 1 curl only, 2 flux only, 3 both).
// Per updated field v (0: E stage / E traces, 1: H stage / H traces) a variant of the
// matrices; they differ only for mixed orders (H ∈ P^{p-1}: B1[0] ignores H's modes
// >= N(p-1) as curl input, B1[1] has no output columns there, B2[1] no rows there).
// Operators B1, B2, Bf, Bb are stored pre-tiled: [n-tile][k-tile][16][BST], BST =
// 96 NH + 4, each tile in the GEMM's shared-memory layout (stage type: the three
// gathered component blocks).
struct DenseOps {
  double *B1[2] = {nullptr, nullptr}, *B2[2] = {nullptr, nullptr}, *AB = nullptr;
  int nc1 = 0, nc2 = 0, k1a = 0;
  int nkt1 = 0, nkt2 = 0, nktf = 0, nktb = 0;   // k-tiles of B1, B2, Bf, Bb (pool strides)
  // warp columns per GEMM CTA (CTA tile = 64 elements x 96 NH columns); the host pads
  // the operator layouts to them. Stage type (B1, Bb): NH = 1 takes the three component
  // blocks of 32 modes, NH = 2 of 64 modes, the warp columns alternating 8-mode groups.
  // Trace type (B2, Bf): contiguous columns, warp columns alternating 8-column groups.
  int stage_nh = 1;
  unsigned long long *tile_ctr = nullptr;   // GEMM dynamic tile counter (null: static tile order)
  int trace_nh = 1;
  uint64_t *ktl1[2][4] = {};
  int32_t *ktoff1[2][4] = {};
  uint64_t *ktl2[2] = {nullptr, nullptr};
  int32_t *ktoff2[2] = {nullptr, nullptr};
  // material points (reverse numerical integration): Bf [3Nk][ncf] residual -> point
  // values, Bb [3Qk][nc1] point values -> modes; SWe/SWm [n][Qk] = ŵ_i / ε, μ at the
  // points; AC [n][3Nk] residual scratch, P [n][3Qk] point-value scratch
  double *Bf = nullptr, *Bb = nullptr, *SWe = nullptr, *SWm = nullptr, *AC = nullptr, *P = nullptr;
  // curved elements: per point K_i = ŵ_i F(ξ_i)ᵀF(ξ_i) / (m det F(ξ_i)), [n][Qk][6] (E: ε, H: μ)
  double *KE = nullptr, *KH = nullptr;
  // sum-factorised point transforms (dgm_sumfact.cu): 1D tables Pc, Bb, Ca, 1/‖φ‖², and
  // the (i, j, k) of every graded mode
  double *sf_tab = nullptr;
  int3 *sf_modes = nullptr;
  int2 *sf_pairs = nullptr;
  int sf_pc = 0, sf_bb = 0, sf_ca = 0, sf_in = 0;   // offsets into sf_tab
  int use_sumfact = 1;                               // 0: dense Φ GEMMs (DGM_POINT_GEMM=1)
  uint64_t *ktlf = nullptr, *ktlb = nullptr;
  int32_t *ktofff = nullptr, *ktoffb = nullptr;
  int ncf = 0;
  // streamed sparse curl (hybrid engine, dgm_curl.cuh): ĉ scratch [3][n_tet][ldc]
  double *Cc = nullptr;
  int ldc = 0;
};


struct DevProgs {
  DevProg curl;
  DevSProg strace[4];
  DevSProg slift[4];
  const double *__restrict__ norms;
};

// Per-element geometry, 80 bytes: G' = FᵀF/det F (symmetric, 6 entries
// g00 g01 g02 g11 g12 g22), det F, 1/ε, 1/μ, Z = sqrt(μ/ε).
struct Geo {
  double g[6];
  double detF, inv_eps, inv_mu, Z;
};

// sum-factorised reverse numerical integration (dgm_sumfact.cu)
struct SumfactArgs {
  const double *AC;       // residual after the reference mass, [n][acld], component c at c*acNk
  int64_t acld;
  int acNk;
  const double *Pc, *Bb, *Ca, *inv_norms;
  const int3 *modes;
  const int2 *pairs;      // the (i, j) with i + j <= p, i outer
  const double *K;        // curved: [n][Qk][6] point factors (else null)
  const double *SW;       // flat variable materials: [n][Qk] ŵ_i / m(x_i)
  int Qk;
  const Geo *geo;
  double *X, *dX;
  double dt;
  int64_t n_tet;
  int LD, stageE, out_mode;
};

enum OutMode { OUT_UPDATE = 0, OUT_WRITE = 1, OUT_ACCUM = 2 };
enum Stage { STAGE_E = 0, STAGE_H = 1 };   // STAGE_E updates E from H (Y=H, X=E)

struct StageArgs {
  const double *Y;       // other field (curl and central-flux source)
  double *X;             // updated field (OUT_UPDATE)
  double *dX;            // derivative output (OUT_WRITE / OUT_ACCUM)
  const double *trX;     // upwind: tangential traces of the updated field (trace-buffer layout)
  const Geo *geo;
  const int32_t *nbr;    // [n][4], -1 PEC
  const int8_t *nbrf;    // [n][4], -1 PEC
  const double *fmet;    // upwind: [n][4][3] M00 M01 M11
  const double *HF;      // stabilised flux, E stage: face unknowns [n_faces][2][NF] (else null)
  const int32_t *fid;    // [n][4] face index
  int64_t n_tet;
  double dt;
  int stage, upwind, do_curl, do_flux, out_mode;
};

}  // namespace dgm

// captured multi-step CUDA graph: valid for these field pointers, dt and the
// trace-buffer parities at the start of a chunk
struct GraphKey {
  const double *E, *H, *HF;
  double dt;
  int ce, ch;
  bool operator==(const GraphKey &o) const {
    return E == o.E && H == o.H && HF == o.HF && dt == o.dt && ce == o.ce && ch == o.ch;
  }
};

struct dgm_ctx {
  int p = 0, N = 0, NF = 0, LD = 0;
  int64_t n_tet = 0;
  int flux = 0;
  int sms = 0;
  int engine = 0;      // 0: sparse recurrence kernels, 1: dense DMMA contractions (DGM_ENGINE=dense)
  int sparse_curl = 0; // engine 1 only: the curl by the streamed recurrence sweeps (hybrid engine)
  int mixed = 0;       // 1: H ∈ P^{p-1} (E ∈ P^p), dense engine only; NH = N(p-1)
  int matq = 0;        // 1: the point pipeline of the inverse mass (material points or curved elements)
  int curved = 0;      // 1: curved (quadratic) elements, per-point 3x3 factors h_ke / h_kh
  int Q = 0, Qk = 0;   // quadrature points per element (collapsed Gauss–Jacobi, q = p+2), padded
  std::vector<double> h_swe, h_swm, h_ke, h_kh;
  int NH = 0;
  dgm::DenseOps dense{};
  void *d_dense = nullptr;
  dgm::DevStream stream{};
  void *d_stream = nullptr;
  int use_graphs = 1;                 // long dgm_step runs replay a captured graph (DGM_GRAPHS=0: off)
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey{};
  int64_t glaunches = 0;              // kernel launches per captured chunk
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev[2] = {nullptr, nullptr};
  std::vector<int32_t> nbr;
  std::vector<int8_t> nbrf, sign, bc;
  std::vector<dgm::Geo> h_geo;
  std::vector<double> h_fmet;
  dgm::Geo *d_geo = nullptr;
  int32_t *d_nbr = nullptr;
  int8_t *d_nbrf = nullptr;
  double *d_fmet = nullptr;
  void *d_blob = nullptr;
  dgm::DevProgs progs{};
  double *d_tr[4] = {nullptr, nullptr, nullptr, nullptr};  // lane path: TE0, TE1, TH0, TH1
  double *d_partial = nullptr; // energy partial sums
  int64_t n_partial = 0;
  double *d_E = nullptr, *d_H = nullptr;   // device copies for dgm_step_host
  double *d_pw[3] = {nullptr, nullptr, nullptr};   // power-iteration work fields
  cudaStream_t side = nullptr;             // dgm_step_host: H copies overlap the kernels
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t launches = 0;
  // stabilised central flux
  int64_t n_faces = 0;
  double alpha = 1.0;
  std::vector<int32_t> fid;            // [n][4]
  std::vector<int32_t> fside;          // [n_faces][2]: 4*tet+face of the two sides (-1: PEC)
  std::vector<double> fgeo;            // [n_faces][8]: Minv00 Minv01 Minv11, h/α, M00 M01 M11, 0
  int32_t *d_fid = nullptr, *d_fside = nullptr;
  int8_t *d_sign = nullptr;
  double *d_fgeo = nullptr, *d_fnorms = nullptr;
  const double *cur_HF = nullptr;      // HF of the running *_sc call
  // trace-buffer state left by the last dgm_step (for DGM_STEP_CONTINUE)
  bool tr_valid = false;
  const double *tr_E = nullptr, *tr_H = nullptr;
  int tr_ce = 0, tr_ch = 0;
  std::string err;
};

namespace dgm {
dgm_status set_err(dgm_ctx *c, dgm_status s, const std::string &msg);
// kernels (dgm_kernels.cu)
// trace-buffer stage scheme for all orders (lane-pair kernels p <= kLanePmax, warp kernels above)
dgm_status launch_tb_stage(dgm_ctx *c, int stage, const double *Y, double *X, double *dX, double dt, int do_curl,
                           int do_flux, int out_mode, const double *trY, const double *trX, double *trOut,
                           cudaStream_t st);
dgm_status launch_tb_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st, int field);   // field: 0 E, 1 H
dgm_status launch_energy(dgm_ctx *c, const double *E, const double *H, double *out_host, cudaStream_t st);
dgm_status launch_hf(dgm_ctx *c, const double *TE, double *HF, double *dHF, double dt, cudaStream_t st);
dgm_status launch_face_energy(dgm_ctx *c, const double *HF, double *out, cudaStream_t st);
dgm_status launch_massdot(dgm_ctx *c, const double *A, const double *B, int use_mu, double *out, cudaStream_t st);
dgm_status launch_scale(dgm_ctx *c, double *X, const double *Y, double s, cudaStream_t st);
dgm_status launch_seed(dgm_ctx *c, double *X, uint64_t seed, cudaStream_t st);
// dense-contraction engine (dgm_dense.cu), all orders
dgm_status launch_dense_stage(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st);
dgm_status launch_dense_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st, int field);
dgm_status launch_sumfact(dgm_ctx *c, const SumfactArgs &a, cudaStream_t st);
// curved elements: P[e][c Qk + i] <- Σ_l K[e][i][c,l] P[e][l Qk + i]
dgm_status launch_pointmix(dgm_ctx *c, double *P, const double *K, cudaStream_t st);
// streamed lane-per-element curl sweeps (dgm_curl.cuh, generated sweep/curl_p*.cu): ĉ of Y
constexpr int kCurlPmin = 4, kCurlPmax = 10;   // orders with generated curl sweeps (hybrid engine)
constexpr int kHybridAuto = 7;                 // AUTO picks the hybrid engine from this order on
dgm_status launch_curl_p4(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl_p5(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl_p6(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl_p7(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl_p8(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl_p9(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
dgm_status launch_curl_p10(dgm_ctx *c, const double *Y, double *C, cudaStream_t st);
// trace buffers use the 16-element interleaved layout only on the sparse lane path
inline bool lane_layout(const dgm_ctx *c);

// streamed-table high-order path (dgm_stream.cu), p > kLanePmax
dgm_status launch_stream_stage(dgm_ctx *c, const StageArgs &a, const double *trY, double *trOut, cudaStream_t st);
dgm_status launch_stream_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st);

// lane-per-element path (dgm_lane.cu), p <= kLanePmax
constexpr int kLanePmax = 6;
dgm_status launch_lane_stage(dgm_ctx *c, int stage, const double *Y, double *X, double *dX, double dt, int do_curl,
                             int do_flux, int out_mode, const double *trY, const double *trX, double *trOut,
                             cudaStream_t st);
dgm_status launch_lane_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st);
}  // namespace dgm

inline bool dgm::lane_layout(const dgm_ctx *c) { return c->engine == 0 && c->p <= dgm::kLanePmax; }
