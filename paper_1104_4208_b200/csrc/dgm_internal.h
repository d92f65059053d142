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
};
struct DevSProg {
  DevProg prog;
  int n_in, n_scr;
  const uint16_t *__restrict__ out;
};
struct DevProgs {
  DevProg curl;
  DevProg trace[4];
  DevProg lift[4];
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

struct dgm_ctx {
  int p = 0, N = 0, NF = 0, LD = 0;
  int64_t n_tet = 0;
  int flux = 0;
  int sms = 0;
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
dgm_status launch_tb_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st);
dgm_status launch_energy(dgm_ctx *c, const double *E, const double *H, double *out_host, cudaStream_t st);
dgm_status launch_hf(dgm_ctx *c, const double *TE, double *HF, double *dHF, double dt, cudaStream_t st);
dgm_status launch_face_energy(dgm_ctx *c, const double *HF, double *out, cudaStream_t st);
dgm_status launch_massdot(dgm_ctx *c, const double *A, const double *B, int use_mu, double *out, cudaStream_t st);
dgm_status launch_scale(dgm_ctx *c, double *X, const double *Y, double s, cudaStream_t st);
dgm_status launch_seed(dgm_ctx *c, double *X, uint64_t seed, cudaStream_t st);
// lane-per-element path (dgm_lane.cu), p <= kLanePmax
constexpr int kLanePmax = 6;
dgm_status launch_lane_stage(dgm_ctx *c, int stage, const double *Y, double *X, double *dX, double dt, int do_curl,
                             int do_flux, int out_mode, const double *trY, const double *trX, double *trOut,
                             cudaStream_t st);
dgm_status launch_lane_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st);
}  // namespace dgm
