// Stage dispatch for all orders and engines (lane-pair p <= kLanePmax, streamed
// tables above, dense engine), the stabilised-flux face kernels, and the reductions
// (energy, mass inner product).  Per element a stage does (SURVEY.md §8(a) S1-S6,
// DESIGN.md §6):
//   S1  reference curl of Ŷ by the sparse recurrence sweeps (level-scheduled
//       pull-form program from gen/plan.py)
//   S3  own and neighbour tangential traces of Ŷ read from the trace buffer
//   S4  numerical flux on the face modes (central or upwind, PEC mirror)
//   S5  lift back to volume modes (sum-factorised staged transpose of the trace,
//       ‖ψ‖²/‖φ‖² folded in)
//   S2  inverse mass + geometry: Ẋ_β = ±(1/m_T) G'_T (ĉ_β + L_β),
//       G'_T = F_TᵀF_T/det F_T (covariant identities :367-370)
//   S6  update X += dt Ẋ (symplectic Euler) or write Ẋ, then
//       the traces of the updated field for the next stage.
#include <cstdint>
#include <cstdio>

#include "dgm_internal.h"

namespace dgm {

// mode counts of order P (graded Dubiner basis, SURVEY.md §8 notation)
template <int P>
struct Dim {
  static constexpr int N = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NF = (P + 1) * (P + 2) / 2;
  static constexpr int LD = (N + 3) & ~3;
};

// Energy ½ Σ_T sgn(det F) Σ_α ‖φ_α‖² (ε Ê_αᵀ G'^{-1} Ê_α + μ Ĥ_αᵀ G'^{-1} Ĥ_α)
// (|det F| F^{-1}F^{-T} = sgn G'^{-1}).  One thread
// per element, fixed grid, per-block partials: deterministic.
template <int P>
__global__ void energy_kernel(const double *__restrict__ E, const double *__restrict__ H, const Geo *__restrict__ geo,
                              const double *__restrict__ norms, int64_t n_tet, double *partial) {
  using D = Dim<P>;
  constexpr int N = D::N, LD = D::LD;
  const int64_t cstride = n_tet * LD;
  double sum = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_tet; e += (int64_t)gridDim.x * blockDim.x) {
    const Geo g = geo[e];
    // inverse of the symmetric G'
    const double a = g.g[0], b = g.g[1], c = g.g[2], d = g.g[3], f = g.g[4], h = g.g[5];
    const double c00 = d * h - f * f, c01 = c * f - b * h, c02 = b * f - c * d;
    const double c11 = a * h - c * c, c12 = b * c - a * f, c22 = a * d - b * b;
    const double det = a * c00 + b * c01 + c * c02;
    const double id = 1.0 / det;
    const double eps = 1.0 / g.inv_eps, mu = 1.0 / g.inv_mu;
    double se = 0.0, sh = 0.0;
    for (int al = 0; al < N; ++al) {
      const int64_t o = e * LD + al;
      const double e0 = E[o], e1 = E[cstride + o], e2 = E[2 * cstride + o];
      const double h0 = H[o], h1 = H[cstride + o], h2 = H[2 * cstride + o];
      const double qe = c00 * e0 * e0 + c11 * e1 * e1 + c22 * e2 * e2 + 2.0 * (c01 * e0 * e1 + c02 * e0 * e2 + c12 * e1 * e2);
      const double qh = c00 * h0 * h0 + c11 * h1 * h1 + c22 * h2 * h2 + 2.0 * (c01 * h0 * h1 + c02 * h0 * h2 + c12 * h1 * h2);
      se += norms[al] * qe;
      sh += norms[al] * qh;
    }
    const double sg = g.detF > 0 ? 1.0 : -1.0;
    sum += 0.5 * sg * id * (eps * se + mu * sh);
  }
  __shared__ double red[256];
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void sum_kernel(const double *partial, int n, double *out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// ---------------------------------------------------------------------------
#define DGM_DISPATCH(p, fn, ...)          \
  switch (p) {                            \
    case 1: return fn<1>(__VA_ARGS__);    \
    case 2: return fn<2>(__VA_ARGS__);    \
    case 3: return fn<3>(__VA_ARGS__);    \
    case 4: return fn<4>(__VA_ARGS__);    \
    case 5: return fn<5>(__VA_ARGS__);    \
    case 6: return fn<6>(__VA_ARGS__);    \
    case 7: return fn<7>(__VA_ARGS__);    \
    case 8: return fn<8>(__VA_ARGS__);    \
    case 9: return fn<9>(__VA_ARGS__);    \
    case 10: return fn<10>(__VA_ARGS__);  \
    default: return DGM_EORDER;           \
  }

dgm_status launch_tb_stage(dgm_ctx *c, int stage, const double *Y, double *X, double *dX, double dt, int do_curl,
                           int do_flux, int out_mode, const double *trY, const double *trX, double *trOut,
                           cudaStream_t st) {
  if (c->n_tet == 0) return DGM_OK;
  if (c->engine == 0 && c->p <= kLanePmax)
    return launch_lane_stage(c, stage, Y, X, dX, dt, do_curl, do_flux, out_mode, trY, trX, trOut, st);
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
  if (c->engine == 1) return launch_dense_stage(c, a, trY, trOut, st);
  return launch_stream_stage(c, a, trY, trOut, st);
}

dgm_status launch_tb_traces(dgm_ctx *c, const double *X, double *tr, cudaStream_t st, int field) {
  if (c->n_tet == 0) return DGM_OK;
  if (c->engine == 1) return launch_dense_traces(c, X, tr, st, field);
  if (c->p <= kLanePmax) return launch_lane_traces(c, X, tr, st);
  return launch_stream_traces(c, X, tr, st);
}

// (A, M_m B) = Σ_T |det F| m_T Σ_α ‖φ_α‖² A_αᵀ F^{-1}F^{-T} B_α  (m = ε or μ), the
// mass inner product of the covariant fields; per-block partials.
template <int P>
__global__ void massdot_kernel(const double *__restrict__ A, const double *__restrict__ B, const Geo *__restrict__ geo,
                               const double *__restrict__ norms, int64_t n_tet, int use_mu, double *partial) {
  using D = Dim<P>;
  constexpr int N = D::N, LD = D::LD;
  const int64_t cstride = n_tet * LD;
  double sum = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_tet; e += (int64_t)gridDim.x * blockDim.x) {
    const Geo g = geo[e];
    const double a = g.g[0], b = g.g[1], c = g.g[2], d = g.g[3], f = g.g[4], h = g.g[5];
    const double c00 = d * h - f * f, c01 = c * f - b * h, c02 = b * f - c * d;
    const double c11 = a * h - c * c, c12 = b * c - a * f, c22 = a * d - b * b;
    const double det = a * c00 + b * c01 + c * c02;
    const double m = use_mu ? 1.0 / g.inv_mu : 1.0 / g.inv_eps;
    double se = 0.0;
    for (int al = 0; al < N; ++al) {
      const int64_t o = e * LD + al;
      const double a0 = A[o], a1 = A[cstride + o], a2 = A[2 * cstride + o];
      const double b0 = B[o], b1 = B[cstride + o], b2 = B[2 * cstride + o];
      const double q = c00 * a0 * b0 + c11 * a1 * b1 + c22 * a2 * b2 + c01 * (a0 * b1 + a1 * b0) +
                       c02 * (a0 * b2 + a2 * b0) + c12 * (a1 * b2 + a2 * b1);
      se += norms[al] * q;
    }
    const double sg = g.detF > 0 ? 1.0 : -1.0;
    sum += sg / det * m * se;
  }
  __shared__ double red[256];
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// X[:, :, :N] = s * Y[:, :, :N] (padding untouched; X == Y allowed)
__global__ void scale_kernel(double *X, const double *Y, double s, int64_t n_tet, int N, int LD) {
  const int64_t total = 3 * n_tet * LD;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    if (i % LD < N) X[i] = s * Y[i];
}

// deterministic start vector for the power iteration: a counter-based hash of the
// index mapped to [-1, 1) (splitmix64), modes damped by 1/(1+mode)
__global__ void seed_kernel(double *X, uint64_t seed, int64_t n_tet, int N, int LD) {
  const int64_t total = 3 * n_tet * LD;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int al = (int)(i % LD);
    if (al >= N) { X[i] = 0.0; continue; }
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    X[i] = ((double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0) / (1.0 + al);
  }
}

// Stabilised central flux, face equation (signs reading G16):
//   Ḣ^F_γ = (α/h_F) M^{-1} Σ_{T∋F} σ_{T,f} (E_2, -E_1)_{T,f,γ}   (face mass h_F/α, reading G17)
// from the tangential traces of E in the trace buffer (both layouts); one thread per
// (face, mode).  HF += dt Ḣ^F (update) or dHF = Ḣ^F (write).
__global__ void hf_kernel(const double *__restrict__ TE, double *HF, double *dHF, double dt,
                          const int32_t *__restrict__ fside, const int8_t *__restrict__ sign,
                          const double *__restrict__ fgeo, int64_t n_faces, int NF, int lane_layout) {
  const int64_t total = n_faces * NF;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / NF;
    const int g = (int)(i - k * NF);
    double r1 = 0.0, r2 = 0.0;
    for (int sd = 0; sd < 2; ++sd) {
      const int32_t tf = fside[2 * k + sd];
      if (tf < 0) continue;
      const int64_t e = tf >> 2;
      const int f = tf & 3;
      int64_t i1, i2;
      if (lane_layout) {
        i1 = (((e >> 4) * 8 * NF + (f * 2 + 0) * NF + g) << 4) + (e & 15);
        i2 = (((e >> 4) * 8 * NF + (f * 2 + 1) * NF + g) << 4) + (e & 15);
      } else {
        i1 = (e * 4 + f) * 2 * NF + g;
        i2 = i1 + NF;
      }
      const double sg = (double)sign[tf];
      r1 += sg * __ldg(TE + i2);
      r2 -= sg * __ldg(TE + i1);
    }
    const double *G = fgeo + 8 * k;
    const double d1 = G[3] * (G[0] * r1 + G[1] * r2);
    const double d2 = G[3] * (G[1] * r1 + G[2] * r2);
    double *o = HF ? HF : dHF;
    const int64_t b = k * 2 * NF + g;
    if (HF) {
      o[b] += dt * d1;
      o[b + NF] += dt * d2;
    } else {
      o[b] = d1;
      o[b + NF] = d2;
    }
  }
}

// ½ Σ_F (h_F/α) Σ_γ ‖ψ_γ‖² H_γᵀ M H_γ  (face part of the stabilised energy; fgeo[3] = α/h_F)
__global__ void face_energy_kernel(const double *__restrict__ HF, const double *__restrict__ fgeo,
                                   const double *__restrict__ fnorms, int64_t n_faces, int NF, double *partial) {
  double sum = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_faces; k += (int64_t)gridDim.x * blockDim.x) {
    const double *G = fgeo + 8 * k;
    double q = 0.0;
    for (int g = 0; g < NF; ++g) {
      const double h1 = HF[k * 2 * NF + g], h2 = HF[k * 2 * NF + NF + g];
      q += fnorms[g] * (G[4] * h1 * h1 + 2.0 * G[5] * h1 * h2 + G[6] * h2 * h2);
    }
    sum += 0.5 / G[3] * q;
  }
  __shared__ double red[256];
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

dgm_status launch_hf(dgm_ctx *c, const double *TE, double *HF, double *dHF, double dt, cudaStream_t st) {
  if (c->n_faces == 0) return DGM_OK;
  const int64_t total = c->n_faces * c->NF;
  int64_t grid = (total + 255) / 256;
  if (grid > 8 * (int64_t)c->sms) grid = 8 * (int64_t)c->sms;
  hf_kernel<<<(unsigned)grid, 256, 0, st>>>(TE, HF, dHF, dt, c->d_fside, c->d_sign, c->d_fgeo, c->n_faces, c->NF,
                                            lane_layout(c) ? 1 : 0);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("hf_kernel: ") + cudaGetErrorString(e));
}

dgm_status launch_face_energy(dgm_ctx *c, const double *HF, double *out, cudaStream_t st) {
  const int threads = 256;
  int64_t grid = (c->n_faces + threads - 1) / threads;
  if (grid > 4 * (int64_t)c->sms) grid = 4 * (int64_t)c->sms;
  if (grid < 1) grid = 1;
  if (c->n_partial < grid + 1) {
    cudaFree(c->d_partial);
    if (cudaMalloc(&c->d_partial, sizeof(double) * (grid + 1)) != cudaSuccess) return set_err(c, DGM_ENOMEM, "partials");
    c->n_partial = grid + 1;
  }
  face_energy_kernel<<<(unsigned)grid, threads, 0, st>>>(HF, c->d_fgeo, c->d_fnorms, c->n_faces, c->NF, c->d_partial);
  sum_kernel<<<1, 256, 0, st>>>(c->d_partial, (int)grid, c->d_partial + grid);
  cudaError_t e = cudaMemcpyAsync(out, c->d_partial + grid, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("face_energy: ") + cudaGetErrorString(e));
}

template <int P>
static dgm_status launch_massdot_p(dgm_ctx *c, const double *A, const double *B, int use_mu, double *out,
                                   cudaStream_t st) {
  const int threads = 256;
  int64_t grid = (c->n_tet + threads - 1) / threads;
  if (grid > 4 * (int64_t)c->sms) grid = 4 * (int64_t)c->sms;
  if (c->n_partial < grid + 1) {
    cudaFree(c->d_partial);
    if (cudaMalloc(&c->d_partial, sizeof(double) * (grid + 1)) != cudaSuccess)
      return set_err(c, DGM_ENOMEM, "partials");
    c->n_partial = grid + 1;
  }
  massdot_kernel<P><<<(unsigned)grid, threads, 0, st>>>(A, B, c->d_geo, c->progs.norms, c->n_tet, use_mu, c->d_partial);
  sum_kernel<<<1, 256, 0, st>>>(c->d_partial, (int)grid, c->d_partial + grid);
  cudaError_t e = cudaMemcpyAsync(out, c->d_partial + grid, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_err(c, DGM_ECUDA, std::string("massdot: ") + cudaGetErrorString(e));
  return DGM_OK;
}

dgm_status launch_massdot(dgm_ctx *c, const double *A, const double *B, int use_mu, double *out, cudaStream_t st) {
  DGM_DISPATCH(c->p, launch_massdot_p, c, A, B, use_mu, out, st)
}

dgm_status launch_scale(dgm_ctx *c, double *X, const double *Y, double s, cudaStream_t st) {
  scale_kernel<<<4 * c->sms, 256, 0, st>>>(X, Y, s, c->n_tet, c->N, c->LD);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("scale: ") + cudaGetErrorString(e));
}

dgm_status launch_seed(dgm_ctx *c, double *X, uint64_t seed, cudaStream_t st) {
  seed_kernel<<<4 * c->sms, 256, 0, st>>>(X, seed, c->n_tet, c->N, c->LD);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DGM_OK : set_err(c, DGM_ECUDA, std::string("seed: ") + cudaGetErrorString(e));
}

template <int P>
static dgm_status launch_energy_p(dgm_ctx *c, const double *E, const double *H, double *out, cudaStream_t st) {
  const int threads = 256;
  int64_t grid = (c->n_tet + threads - 1) / threads;
  if (grid > 4 * (int64_t)c->sms) grid = 4 * (int64_t)c->sms;
  if (c->n_partial < grid + 1) {
    cudaFree(c->d_partial);
    if (cudaMalloc(&c->d_partial, sizeof(double) * (grid + 1)) != cudaSuccess)
      return set_err(c, DGM_ENOMEM, "energy partials");
    c->n_partial = grid + 1;
  }
  energy_kernel<P><<<(unsigned)grid, threads, 0, st>>>(E, H, c->d_geo, c->progs.norms, c->n_tet, c->d_partial);
  sum_kernel<<<1, 256, 0, st>>>(c->d_partial, (int)grid, c->d_partial + grid);
  cudaError_t e = cudaMemcpyAsync(out, c->d_partial + grid, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_err(c, DGM_ECUDA, std::string("energy: ") + cudaGetErrorString(e));
  return DGM_OK;
}

dgm_status launch_energy(dgm_ctx *c, const double *E, const double *H, double *out, cudaStream_t st) {
  DGM_DISPATCH(c->p, launch_energy_p, c, E, H, out, st)
}


}  // namespace dgm
