// Host side of the C ABI: mesh validation, face matching, geometry, program
// upload and the call wrappers (SURVEY.md §3 call stacks 1-4).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include "dgm_internal.h"

using dgm::Geo;
using dgm::HostProg;
using dgm::HostProgSet;

#include "generated_tables.inc"

static thread_local std::string g_create_err;  // message of the last failed dgm_create

namespace dgm {

dgm_status set_err(dgm_ctx *c, dgm_status s, const std::string &msg) {
  if (c) c->err = msg;
  return s;
}

}  // namespace dgm

namespace {

#define CUDA_TRY(ctx, call)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return dgm::set_err(ctx, e_ == cudaErrorMemoryAllocation ? DGM_ENOMEM : DGM_ECUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));           \
  } while (0)

struct FaceRec {
  int32_t r[3];
  int32_t tet;
  int8_t f;
};

// Face f of a tet is opposite local vertex f; its vertices are the other three
// in ascending local order (= ascending representative order; reading G9).
const int kFaceVerts[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

size_t prog_bytes(const HostProg &p) {
  size_t rows = (size_t)p.npass * 32, terms = (size_t)p.nterm * 32;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(rows * 2) * 2 + al(terms * 2) + al(terms * 8) + al((p.npass + 1) * 4) + al(p.npass + 1) + al(terms * 16) +
         al(rows * 8) + al((p.npass + 1) * 8);
}

// Copy one program into the staging buffer at *off, return its device view.
dgm::DevProg stage_prog(const HostProg &p, std::vector<char> &buf, size_t &off, char *dev_base) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  auto put = [&](const void *src, size_t bytes) -> char * {
    char *d = dev_base + off;
    if (bytes) std::memcpy(buf.data() + off, src, bytes);
    off += al(bytes);
    return d;
  };
  size_t rows = (size_t)p.npass * 32, terms = (size_t)p.nterm * 32;
  dgm::DevProg d;
  d.npass = p.npass;
  d.dst = (const uint16_t *)put(p.dst, rows * 2);
  d.cnt = (const uint16_t *)put(p.cnt, rows * 2);
  d.src = (const uint16_t *)put(p.src, terms * 2);
  d.coef = (const double *)put(p.coef, terms * 8);
  d.off = (const int32_t *)put(p.off, (p.npass + 1) * 4);
  d.sync = (const uint8_t *)put(p.sync, p.npass ? p.npass : 1);
  std::vector<double> packed(terms * 2);
  for (size_t q = 0; q < terms; ++q) {
    packed[2 * q] = p.coef[q];
    long long sv = p.src[q];
    std::memcpy(&packed[2 * q + 1], &sv, 8);
  }
  d.term = (const double2 *)put(packed.data(), terms * 16);
  std::vector<uint32_t> meta(rows * 2);
  for (size_t r = 0; r < rows; ++r) {
    meta[2 * r] = (uint32_t)p.dst[r] | ((uint32_t)p.cnt[r] << 16);
    meta[2 * r + 1] = (uint32_t)(p.off[r / 32] * 32 + (int)(r % 32));
  }
  d.meta = (const uint2 *)put(meta.data(), rows * 8);
  std::vector<int32_t> lv;
  for (int q = 0, ps = 0; q < p.npass; ++q)
    if (p.sync[q]) {
      lv.push_back(ps);
      lv.push_back(q);
      ps = q + 1;
    }
  d.nlev = (int)lv.size() / 2;
  d.lvl = (const int2 *)put(lv.data(), lv.size() * 4);
  return d;
}

// Cut the high-order programs into chunks of whole passes (≤ chunk_cap bytes unless
// one pass is larger) in execution order: curl, slift[0..3], strace[0..3].
dgm_status build_stream(dgm_ctx *c, const HostProgSet &hs, size_t chunk_cap) {
  const HostProg *progs[9] = {&hs.curl,          &hs.slift[0].prog,  &hs.slift[1].prog,
                              &hs.slift[2].prog, &hs.slift[3].prog,  &hs.strace[0].prog,
                              &hs.strace[1].prog, &hs.strace[2].prog, &hs.strace[3].prog};
  std::vector<char> blob;
  std::vector<dgm::StreamChunk> ch;
  dgm::DevStream ds{};
  size_t maxb = 0;
  for (int pi = 0; pi < 9; ++pi) {
    const HostProg &hp = *progs[pi];
    ds.first[pi] = (int)ch.size();
    int q = 0;
    while (q < hp.npass) {
      const int qa = q;
      size_t tb = 0;
      while (q < hp.npass) {
        const size_t w = (size_t)(hp.off[q + 1] - hp.off[q]);
        const size_t nb = 256 * (size_t)(q - qa + 1) + 512 * (tb + w);
        if (q > qa && nb > chunk_cap) break;
        tb += w;
        ++q;
      }
      const int np = q - qa;
      const size_t bytes = 256 * (size_t)np + 512 * tb;
      dgm::StreamChunk sc{(uint32_t)blob.size(), (uint32_t)bytes, np, 0};
      blob.resize(blob.size() + bytes);
      uint32_t *meta = (uint32_t *)(blob.data() + sc.off);
      double *terms = (double *)(blob.data() + sc.off + 256 * (size_t)np);
      size_t base = 0;
      for (int qq = qa; qq < q; ++qq) {
        const int w = hp.off[qq + 1] - hp.off[qq];
        // padded terms (t >= cnt) keep coef 0 but read a slot some real term of this
        // pass reads, so they never touch an unwritten (possibly non-finite) slot
        long long fallback = 0;
        for (int l = 0; l < 32; ++l)
          if (hp.dst[(size_t)qq * 32 + l] != 0xFFFF && hp.cnt[(size_t)qq * 32 + l] > 0) {
            fallback = hp.src[(size_t)hp.off[qq] * 32 + l];
            break;
          }
        for (int l = 0; l < 32; ++l) {
          const size_t r = (size_t)qq * 32 + l;
          meta[2 * ((qq - qa) * 32 + l)] =
              (uint32_t)hp.dst[r] | ((uint32_t)w << 16) | (hp.sync[qq] ? 0x80000000u : 0u);   // uniform pass width
          meta[2 * ((qq - qa) * 32 + l) + 1] = (uint32_t)(base + l);
          for (int t = 0; t < w; ++t) {
            const size_t gi = ((size_t)hp.off[qq] + t) * 32 + l;
            const size_t li = base + (size_t)t * 32 + l;
            const bool real = hp.dst[r] != 0xFFFF && t < hp.cnt[r];
            terms[2 * li] = real ? hp.coef[gi] : 0.0;
            long long sv = real ? (long long)hp.src[gi] : fallback;
            std::memcpy(&terms[2 * li + 1], &sv, 8);
          }
        }
        base += (size_t)w * 32;
      }
      ch.push_back(sc);
      if (bytes > maxb) maxb = bytes;
    }
    ds.count[pi] = (int)ch.size() - ds.first[pi];
  }
  ds.nchunk = (int)ch.size();
  ds.max_bytes = (int)((maxb + 127) & ~size_t(127));
  const size_t cb = (ch.size() * sizeof(dgm::StreamChunk) + 255) & ~size_t(255);
  CUDA_TRY(c, cudaMalloc(&c->d_stream, cb + blob.size()));
  CUDA_TRY(c, cudaMemcpy(c->d_stream, ch.data(), ch.size() * sizeof(dgm::StreamChunk), cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy((char *)c->d_stream + cb, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  ds.chunks = (const dgm::StreamChunk *)c->d_stream;
  ds.base = (const char *)c->d_stream + cb;
  c->stream = ds;
  return DGM_OK;
}

// ---- reverse numerical integration (variable materials inside elements) -------
// Jacobi P_n^{(a,0)}(x) and its derivative by the three-term recurrence.
void jacobi_pd(int n, double a, double x, double &P, double &dP) {
  double p0 = 1.0, p1 = 0.5 * (a + (a + 2.0) * x);   // P_1^{(a,0)} = (a + (a+2) x)/2
  double d0 = 0.0, d1 = 0.5 * (a + 2.0);
  if (n == 0) {
    P = 1.0;
    dP = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const double kk = k, c = 2.0 * kk + a;
    const double A = 2.0 * kk * (kk + a) * (c - 2.0);
    const double B = (c - 1.0) * (c * (c - 2.0) * x + a * a);
    const double C = 2.0 * (kk + a - 1.0) * (kk - 1.0) * c;
    const double p2 = (B * p1 - C * p0) / A;
    const double d2 = (B * d1 + (c - 1.0) * c * (c - 2.0) * p1 - C * d0) / A;
    p0 = p1;
    p1 = p2;
    d0 = d1;
    d1 = d2;
  }
  P = p1;
  dP = d1;
}
// q-point Gauss–Jacobi rule for the weight (1-x)^a on [-1,1]: Newton on the zeros of
// P_q^{(a,0)} with deflation, weights 2^{a+1} / ((1-x²) P'(x)²).
void gauss_jacobi(int q, double a, std::vector<double> &x, std::vector<double> &w) {
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  for (int k = 0; k < q; ++k) {
    double r = -std::cos((2.0 * k + 1.0) * M_PI / (2.0 * q));   // Chebyshev guess
    if (k > 0) r = 0.5 * (r + x[k - 1]);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      jacobi_pd(q, a, r, P, dP);
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += 1.0 / (r - x[i]);
      const double delta = -P / (dP - s * P);
      r += delta;
      if (std::fabs(delta) < 1e-16) break;
    }
    x[k] = r;
  }
  for (int k = 0; k < q; ++k) {
    double P, dP;
    jacobi_pd(q, a, x[k], P, dP);
    w[k] = std::pow(2.0, a + 1.0) / ((1.0 - x[k] * x[k]) * dP * dP);
  }
}
// Collapsed rule on the reference tet (q = p+2 per direction, exact to degree 2q-1):
// x = (1+a)/2, y = (1-a)(1+b)/4, z = (1-a)(1-b)(1+c)/8, weights (2,0),(1,0),(0,0) / 64.
void tet_quadrature(int p, std::vector<double> &xi, std::vector<double> &w) {
  const int q = p + 2;
  std::vector<double> a, wa, b, wb, c, wc;
  gauss_jacobi(q, 2.0, a, wa);
  gauss_jacobi(q, 1.0, b, wb);
  gauss_jacobi(q, 0.0, c, wc);
  xi.clear();
  w.clear();
  for (int i = 0; i < q; ++i)
    for (int j = 0; j < q; ++j)
      for (int k = 0; k < q; ++k) {
        xi.push_back(0.5 * (1.0 + a[i]));
        xi.push_back(0.25 * (1.0 - a[i]) * (1.0 + b[j]));
        xi.push_back(0.125 * (1.0 - a[i]) * (1.0 - b[j]) * (1.0 + c[k]));
        w.push_back(wa[i] * wb[j] * wc[k] / 64.0);
      }
}
// φ_ijk(x,y,z) = (1-x-y)^i (1-x)^j P_i(2z/(1-x-y)-1) P_j^{(2i+1,0)}(2y/(1-x)-1)
//               P_k^{(2i+2j+2,0)}(2x-1), graded ABI mode order.
void basis_at(int p, const double *pt, double *out) {
  const double x = pt[0], y = pt[1], z = pt[2];
  const double s = 1.0 - x - y, r = 1.0 - x;
  int m = 0;
  for (int n = 0; n <= p; ++n)
    for (int i = 0; i <= n; ++i)
      for (int j = 0; j <= n - i; ++j) {
        const int k = n - i - j;
        double Pi, Pj, Pk, d;
        jacobi_pd(i, 0.0, 2.0 * z / s - 1.0, Pi, d);
        jacobi_pd(j, 2.0 * i + 1.0, 2.0 * y / r - 1.0, Pj, d);
        jacobi_pd(k, 2.0 * i + 2.0 * j + 2.0, 2.0 * x - 1.0, Pk, d);
        out[m++] = std::pow(s, i) * std::pow(r, j) * Pi * Pj * Pk;
      }
}

// ---- dense engine: assemble the operator matrices from the exact programs ------
// Scalar executor of an ELL program (passes in order respect the DAG levels).
void exec_prog_host(const HostProg &hp, std::vector<double> &s) {
  for (int q = 0; q < hp.npass; ++q)
    for (int l = 0; l < 32; ++l) {
      const size_t r = (size_t)q * 32 + l;
      if (hp.dst[r] == 0xFFFF) continue;
      double acc = 0.0;
      for (int t = 0; t < hp.cnt[r]; ++t) {
        const size_t gi = ((size_t)hp.off[q] + t) * 32 + l;
        acc += hp.coef[gi] * s[hp.src[gi]];
      }
      s[hp.dst[r]] = acc;
    }
}
// Staged program: the first level reads in[], later levels the scratch; returns the
// value of output i (0 when the output has no slot).
void exec_staged_host(const dgm::HostSProg &sp, const std::vector<double> &in, std::vector<double> &scr,
                      std::vector<double> &out, int nout) {
  const HostProg &hp = sp.prog;
  scr.assign(sp.n_scr + 1, 0.0);
  bool first = true;
  for (int q = 0; q < hp.npass; ++q) {
    for (int l = 0; l < 32; ++l) {
      const size_t r = (size_t)q * 32 + l;
      if (hp.dst[r] == 0xFFFF) continue;
      double acc = 0.0;
      for (int t = 0; t < hp.cnt[r]; ++t) {
        const size_t gi = ((size_t)hp.off[q] + t) * 32 + l;
        acc += hp.coef[gi] * (first ? in[hp.src[gi]] : scr[hp.src[gi]]);
      }
      scr[hp.dst[r]] = acc;
    }
    if (hp.sync[q]) first = false;
  }
  out.assign(nout, 0.0);
  for (int i = 0; i < nout; ++i) out[i] = sp.out[i] == 0xFFFF ? 0.0 : scr[sp.out[i]];
}

int64_t n_or1(const dgm_ctx *c) { return c->n_tet > 0 ? c->n_tet : 1; }

dgm_status dense_build(dgm_ctx *c, const HostProgSet &hs) {
  constexpr int BK = 16, BN = 96;
  static const double T1[4][3] = {{-1, 1, 0}, {0, 1, 0}, {1, 0, 0}, {1, 0, 0}};
  static const double T2[4][3] = {{-1, 0, 1}, {0, 0, 1}, {0, 0, 1}, {0, 1, 0}};
  const int N = c->N, NF = c->NF;
  // one warp column for every GEMM: with the dynamic tile order the CTAs of one m-tile
  // share its A rows in L2, and two warp columns (one A tile for 192 columns) measured
  // slower at every order; the overrides keep both layouts testable
  c->dense.stage_nh = 1;
  if (const char *v = std::getenv("DGM_STAGE_NH"))   // measurement override (1 or 2)
    if (std::atoi(v) == 1 || std::atoi(v) == 2) c->dense.stage_nh = std::atoi(v);
  const int NH = c->dense.stage_nh, BNT = BN * NH;
  c->dense.trace_nh = 1;
  if (const char *v = std::getenv("DGM_TRACE_NH"))   // measurement override (1 or 2)
    if (std::atoi(v) == 1 || std::atoi(v) == 2) c->dense.trace_nh = std::atoi(v);
  const int BNT2 = BN * c->dense.trace_nh;
  const int Nk = (N + BK - 1) / BK * BK, NFk = (NF + BK - 1) / BK * BK, Np = (N + 32 * NH - 1) / (32 * NH) * (32 * NH);
  const int k1a = 3 * Nk;
  const int K1 = k1a + 8 * NFk;
  const int K2 = 3 * Nk;
  const int nc1 = 3 * Np;
  const int nc2 = (8 * NF + BNT2 - 1) / BNT2 * BNT2;
  std::vector<double> B1((size_t)K1 * nc1, 0.0), B2((size_t)K2 * nc2, 0.0);
  // curl: column (c, β) of Ĉ by running the sweep program on that unit input
  int maxslot = 0;
  for (int r = 0; r < hs.curl.npass * 32; ++r)
    if (hs.curl.dst[r] != 0xFFFF && hs.curl.dst[r] > maxslot) maxslot = hs.curl.dst[r];
  std::vector<double> sl(std::max(maxslot + 1, 12 * N));
  for (int k = 0; k < 3 * N; ++k) {
    std::fill(sl.begin(), sl.end(), 0.0);
    sl[k] = 1.0;
    exec_prog_host(hs.curl, sl);
    const size_t row = (size_t)(k / N) * Nk + k % N;
    for (int m = 0; m < 3; ++m)
      for (int b = 0; b < N; ++b) B1[row * nc1 + (size_t)m * Np + b] = sl[(size_t)hs.acc + m * N + b];
  }
  // lift: L_f e_γ, spread to the components with t̂1 (A) / t̂2 (B)
  std::vector<double> in, scr, out;
  for (int f = 0; f < 4; ++f)
    for (int g = 0; g < NF; ++g) {
      in.assign(NF, 0.0);
      in[g] = 1.0;
      exec_staged_host(hs.slift[f], in, scr, out, N);
      const size_t ra = (size_t)k1a + (2 * f) * NFk + g, rb = (size_t)k1a + (2 * f + 1) * NFk + g;
      for (int m = 0; m < 3; ++m)
        for (int b = 0; b < N; ++b) {
          B1[ra * nc1 + (size_t)m * Np + b] = T1[f][m] * out[b];
          B1[rb * nc1 + (size_t)m * Np + b] = T2[f][m] * out[b];
        }
    }
  // traces: R_f e_β, tangential weights t̂1 / t̂2 per component
  for (int f = 0; f < 4; ++f)
    for (int b = 0; b < N; ++b) {
      in.assign(N, 0.0);
      in[b] = 1.0;
      exec_staged_host(hs.strace[f], in, scr, out, NF);
      for (int cc = 0; cc < 3; ++cc)
        for (int g = 0; g < NF; ++g) {
          B2[(size_t)(cc * Nk + b) * nc2 + (2 * f) * NF + g] = T1[f][cc] * out[g];
          B2[(size_t)(cc * Nk + b) * nc2 + (2 * f + 1) * NF + g] = T2[f][cc] * out[g];
        }
    }
  // Entries that are exactly zero in the exact operator can come out as rounding
  // residue (~1e-17) of cancelling recurrence terms; clear them so the tile masks see
  // the true sparsity (changes results by < 1e-14 relative).
  auto clean = [](std::vector<double> &B) {
    double mx = 0.0;
    for (double v : B) mx = std::max(mx, std::fabs(v));
    for (double &v : B)
      if (std::fabs(v) <= 1e-13 * mx) v = 0.0;
  };
  clean(B1);
  clean(B2);
  // operator column of CTA-tile column tc (warp column h = tc / 96) of n-tile t.
  // Stage type (gather): the three component blocks of the tile's 32 nh modes, the warp
  // columns taking alternate 8-mode groups (nh = 2).
  // Trace type: the warp columns take the tile's 8-column groups alternately, so both
  // see the same mix of dense and sparse output columns (the per-face trace operators
  // differ a lot in density; contiguous halves left one warp column with 2-3x the
  // blocks of the other at p >= 8)
  auto tile_col = [&](int t, int tc, bool gather, int bnt) {
    const int nh = bnt / BN, h = tc / BN, t3 = tc % BN;
    const int lm = t3 % 32;   // stage type: mode of the warp column; tile mode (lm/8 nh + h) 8 + lm%8
    return gather ? (t3 / 32) * Np + 32 * nh * t + ((lm / 8) * nh + h) * 8 + lm % 8
                  : t * bnt + ((t3 / 8) * nh + h) * 8 + t3 % 8;
  };
  // per n-tile: non-zero k-tiles with the mask of non-zero 16x8 column groups
  constexpr int GW = 8;   // 16x8 blocks (one MMA column group); 12 mask bits per k-tile
  auto tiles = [&](const std::vector<double> &B, int nc, int ntn, bool gather, int klo, int khi,
                   std::vector<uint64_t> &ktl, std::vector<int32_t> &ktoff, int bnt_arg = 0) {
    ktl.clear();
    ktoff.assign(1, 0);
    const int bnt = bnt_arg > 0 ? bnt_arg : BNT;
    for (int t = 0; t < ntn; ++t) {
      for (int kt = klo / BK; kt < khi / BK; ++kt) {
        uint32_t mask = 0;   // 12 bits per warp column: its non-zero 16x8 groups
        for (int grp = 0; grp < bnt / GW; ++grp)
          for (int cc = 0; cc < GW && !(mask >> grp & 1); ++cc) {
            const int tc = grp * GW + cc;   // column within the CTA tile; warp column h = tc / 96
            const int col = tile_col(t, tc, gather, bnt);
            for (int k = kt * BK; k < (kt + 1) * BK; ++k)
              if (B[(size_t)k * nc + col] != 0.0) {
                mask |= 1u << grp;
                break;
              }
          }
        if (mask) ktl.push_back((uint64_t)kt | ((uint64_t)mask << 16));   // kt < 65536
      }
      ktoff.push_back((int32_t)ktl.size());
    }
  };
  // pre-tiled operator pool [n-tile][k-tile][BK][bnt + 4]: every (n-tile, k-tile) tile
  // in the GEMM's shared-memory layout (same columns as `tiles`: tile_col), so a k-tile
  // load is one linear copy
  auto pool = [&](const std::vector<double> &B, int nc, int ntn, bool gather, int bnt) {
    const int bst = bnt + 4, nkt = (int)(B.size() / nc) / BK;
    std::vector<double> P((size_t)ntn * nkt * BK * bst, 0.0);
    for (int t = 0; t < ntn; ++t)
      for (int kt = 0; kt < nkt; ++kt)
        for (int r = 0; r < BK; ++r)
          for (int tc = 0; tc < bnt; ++tc) {
            const int col = tile_col(t, tc, gather, bnt);
            P[(((size_t)t * nkt + kt) * BK + r) * bst + tc] = B[(size_t)(kt * BK + r) * nc + col];
          }
    return P;
  };
  // variants per updated field (0: E, 1: H); mixed orders (H ∈ P^{p-1}, NH = N(p-1)):
  // the E stage ignores H's modes >= NH as curl input, the H stage has no outputs
  // there, and H's traces ignore them (face modes > p of the lift/trace vanish exactly
  // for volume modes of degree <= p-1, so nothing else changes)
  std::vector<double> B1v[2], B2v[2];
  const int nvar = c->mixed ? 2 : 1;
  B1v[0] = B1;
  B2v[0] = B2;
  if (c->mixed) {
    const int NHm = c->NH;
    B1v[1] = B1;
    B2v[1] = B2;
    for (int cc = 0; cc < 3; ++cc)
      for (int b = NHm; b < N; ++b) {
        std::fill_n(&B1v[0][(size_t)(cc * Nk + b) * nc1], nc1, 0.0);   // H as curl input
        std::fill_n(&B2v[1][(size_t)(cc * Nk + b) * nc2], nc2, 0.0);   // H traces
      }
    for (size_t k = 0; k < (size_t)K1; ++k)
      for (int m = 0; m < 3; ++m)
        for (int b = NHm; b < Np; ++b) B1v[1][k * nc1 + (size_t)m * Np + b] = 0.0;   // H outputs
  }
  std::vector<uint64_t> l1[2][4], l2[2];
  std::vector<int32_t> o1[2][4], o2[2];
  for (int v = 0; v < nvar; ++v) {
    tiles(B1v[v], nc1, Np / (32 * NH), true, 0, 0, l1[v][0], o1[v][0]);   // none (sparse curl only)
    tiles(B1v[v], nc1, Np / (32 * NH), true, 0, k1a, l1[v][1], o1[v][1]);
    tiles(B1v[v], nc1, Np / (32 * NH), true, k1a, K1, l1[v][2], o1[v][2]);
    tiles(B1v[v], nc1, Np / (32 * NH), true, 0, K1, l1[v][3], o1[v][3]);
    tiles(B2v[v], nc2, nc2 / BNT2, false, 0, K2, l2[v], o2[v], BNT2);
  }
  if (std::getenv("DGM_DEBUG_DENSE")) {
    auto bits = [](const std::vector<uint64_t> &l) {
      long n = 0;
      for (uint64_t x : l) n += __builtin_popcountll(x >> 16);
      return n;
    };
    std::fprintf(stderr, "dense_build p=%d: B1 %zu k-tiles %ld blocks, B2 %zu k-tiles %ld blocks (16x8)\n", c->p,
                 l1[0][3].size(), bits(l1[0][3]), l2[0].size(), bits(l2[0]));
    // per trace n-tile: k-tiles and 16x8 blocks of each warp column (load balance)
    for (size_t t = 0; t + 1 < o2[0].size(); ++t) {
      long w0 = 0, w1 = 0;
      for (int i = o2[0][t]; i < o2[0][t + 1]; ++i) {
        w0 += __builtin_popcountll((l2[0][i] >> 16) & 0xFFFu);
        w1 += __builtin_popcountll((l2[0][i] >> 28) & 0xFFFu);
      }
      std::fprintf(stderr, "  B2 n-tile %zu: %d k-tiles, blocks %ld | %ld\n", t, o2[0][t + 1] - o2[0][t], w0, w1);
    }
  }
  std::vector<double> P1[2], P2[2];
  for (int v = 0; v < nvar; ++v) {
    P1[v] = pool(B1v[v], nc1, Np / (32 * NH), true, BNT);
    P2[v] = pool(B2v[v], nc2, nc2 / BNT2, false, BNT2);
  }
  // one device allocation
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t bytes = 0;
  for (int v = 0; v < nvar; ++v) {
    bytes += al(P1[v].size() * 8) + al(P2[v].size() * 8) + al(l2[v].size() * 8 + 4) + al(o2[v].size() * 4 + 4);
    for (int i = 0; i < 4; ++i) bytes += al(l1[v][i].size() * 8 + 4) + al(o1[v][i].size() * 4 + 4);
  }
  CUDA_TRY(c, cudaMalloc(&c->d_dense, bytes));
  char *base = (char *)c->d_dense;
  size_t off = 0;
  bool ok = true;
  auto put = [&](const void *src, size_t b) -> char * {
    char *d = base + off;
    if (b && cudaMemcpy(d, src, b, cudaMemcpyHostToDevice) != cudaSuccess) ok = false;
    off += al(b + (b == 0 ? 4 : 0));
    return d;
  };
  dgm::DenseOps &D = c->dense;
  for (int v = 0; v < nvar; ++v) {
    D.B1[v] = (double *)put(P1[v].data(), P1[v].size() * 8);
    D.B2[v] = (double *)put(P2[v].data(), P2[v].size() * 8);
    for (int i = 0; i < 4; ++i) {
      D.ktl1[v][i] = (uint64_t *)put(l1[v][i].data(), l1[v][i].size() * 8);
      D.ktoff1[v][i] = (int32_t *)put(o1[v][i].data(), o1[v][i].size() * 4);
    }
    D.ktl2[v] = (uint64_t *)put(l2[v].data(), l2[v].size() * 8);
    D.ktoff2[v] = (int32_t *)put(o2[v].data(), o2[v].size() * 4);
  }
  if (!ok) return dgm::set_err(c, DGM_ECUDA, "dense_build: upload failed");
  if (nvar == 1) {   // equal orders: both fields use the same operators
    D.B1[1] = D.B1[0];
    D.B2[1] = D.B2[0];
    for (int i = 0; i < 4; ++i) {
      D.ktl1[1][i] = D.ktl1[0][i];
      D.ktoff1[1][i] = D.ktoff1[0][i];
    }
    D.ktl2[1] = D.ktl2[0];
    D.ktoff2[1] = D.ktoff2[0];
  }
  D.nc1 = nc1;
  D.nc2 = nc2;
  D.k1a = k1a;
  D.nkt1 = K1 / BK;
  D.nkt2 = K2 / BK;
  if (c->matq) {
    // reverse numerical integration: residual (component-blocked, Nk rows) -> point
    // values (Qk per component) -> weighted by ŵ_i/m(x_i) -> back to modes with
    // 1/‖φ‖², columns in the B1 output layout m*Np + β
    const int Q = c->Q, Qk = c->Qk;
    std::vector<double> xi, w;
    tet_quadrature(c->p, xi, w);
    std::vector<double> Phi((size_t)Q * N);
    for (int i = 0; i < Q; ++i) basis_at(c->p, &xi[3 * i], &Phi[(size_t)i * N]);
    const int ncf = (3 * Qk + BNT2 - 1) / BNT2 * BNT2;
    std::vector<double> Bf((size_t)3 * Nk * ncf, 0.0), Bb((size_t)3 * Qk * nc1, 0.0);
    for (int cc = 0; cc < 3; ++cc)
      for (int b = 0; b < N; ++b)
        for (int i = 0; i < Q; ++i) {
          Bf[(size_t)(cc * Nk + b) * ncf + cc * Qk + i] = Phi[(size_t)i * N + b];
          Bb[(size_t)(cc * Qk + i) * nc1 + (size_t)cc * Np + b] = Phi[(size_t)i * N + b] / hs.norms[b];
        }
    std::vector<uint64_t> lf, lb;
    std::vector<int32_t> of, ob;
    tiles(Bf, ncf, ncf / BNT2, false, 0, 3 * Nk, lf, of, BNT2);
    tiles(Bb, nc1, Np / (32 * NH), true, 0, 3 * Qk, lb, ob);
    auto up = [&](void **dst, const void *src, size_t b) -> bool {
      if (cudaMalloc(dst, b ? b : 4) != cudaSuccess) return false;
      return !b || cudaMemcpy(*dst, src, b, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    const std::vector<double> Pf = pool(Bf, ncf, ncf / BNT2, false, BNT2), Pb = pool(Bb, nc1, Np / (32 * NH), true, BNT);
    D.nktf = 3 * Nk / BK;
    D.nktb = 3 * Qk / BK;
    bool okm = up((void **)&D.Bf, Pf.data(), Pf.size() * 8) && up((void **)&D.Bb, Pb.data(), Pb.size() * 8) &&
               up((void **)&D.ktlf, lf.data(), lf.size() * 8) && up((void **)&D.ktofff, of.data(), of.size() * 4) &&
               up((void **)&D.ktlb, lb.data(), lb.size() * 8) && up((void **)&D.ktoffb, ob.data(), ob.size() * 4) &&
               up((void **)&D.SWe, c->h_swe.data(), c->h_swe.size() * 8) &&
               up((void **)&D.SWm, c->h_swm.data(), c->h_swm.size() * 8) &&
               (!c->curved || (up((void **)&D.KE, c->h_ke.data(), c->h_ke.size() * 8) &&
                               up((void **)&D.KH, c->h_kh.data(), c->h_kh.size() * 8)));
    if (!okm) return dgm::set_err(c, DGM_ENOMEM, "dense_build: material-point operators");
    // sum-factorised transforms: the 1D factors of φ_ijk at the
    // collapsed rule's coordinates a (x-direction, weight (2,0)), b ((1,0)), c ((0,0)):
    //   Pc[i][γ] = P_i(c_γ),  Bb[i][j][β] = ((1-b_β)/2)^i P_j^{(2i+1,0)}(b_β),
    //   Ca[t][k][α] = ((1-a_α)/2)^t P_k^{(2t+2,0)}(a_α)
    {
      const int p = c->p, P1 = p + 1, q = p + 2;
      std::vector<double> qa, wa, qb, wb, qc, wc;
      gauss_jacobi(q, 2.0, qa, wa);
      gauss_jacobi(q, 1.0, qb, wb);
      gauss_jacobi(q, 0.0, qc, wc);
      D.sf_pc = 0;
      D.sf_bb = P1 * q;
      D.sf_ca = D.sf_bb + P1 * P1 * q;
      D.sf_in = D.sf_ca + P1 * P1 * q;
      std::vector<double> tab((size_t)D.sf_in + N, 0.0);
      double Pv, d;
      for (int i = 0; i <= p; ++i)
        for (int g = 0; g < q; ++g) {
          jacobi_pd(i, 0.0, qc[g], Pv, d);
          tab[D.sf_pc + i * q + g] = Pv;
        }
      for (int i = 0; i <= p; ++i)
        for (int j = 0; i + j <= p; ++j)
          for (int g = 0; g < q; ++g) {
            jacobi_pd(j, 2.0 * i + 1.0, qb[g], Pv, d);
            tab[D.sf_bb + (i * P1 + j) * q + g] = std::pow(0.5 * (1.0 - qb[g]), i) * Pv;
          }
      for (int t = 0; t <= p; ++t)
        for (int k = 0; t + k <= p; ++k)
          for (int g = 0; g < q; ++g) {
            jacobi_pd(k, 2.0 * t + 2.0, qa[g], Pv, d);
            tab[D.sf_ca + (t * P1 + k) * q + g] = std::pow(0.5 * (1.0 - qa[g]), t) * Pv;
          }
      std::vector<int3> modes;
      for (int n = 0; n <= p; ++n)
        for (int i = 0; i <= n; ++i)
          for (int j = 0; j <= n - i; ++j) modes.push_back(make_int3(i, j, n - i - j));
      for (int b = 0; b < N; ++b) tab[D.sf_in + b] = 1.0 / hs.norms[b];
      std::vector<int2> pairs;
      for (int i = 0; i <= p; ++i)
        for (int j = 0; i + j <= p; ++j) pairs.push_back(make_int2(i, j));
      if (!up((void **)&D.sf_tab, tab.data(), tab.size() * 8) ||
          !up((void **)&D.sf_modes, modes.data(), modes.size() * sizeof(int3)) ||
          !up((void **)&D.sf_pairs, pairs.data(), pairs.size() * sizeof(int2)))
        return dgm::set_err(c, DGM_ENOMEM, "dense_build: sum-factorisation tables");
      if (const char *v = std::getenv("DGM_POINT_GEMM")) D.use_sumfact = std::atoi(v) == 0;
    }
    D.ncf = ncf;
    CUDA_TRY(c, cudaMalloc(&D.AC, sizeof(double) * 3 * (size_t)Nk * (size_t)(n_or1(c))));
    CUDA_TRY(c, cudaMemset(D.AC, 0, sizeof(double) * 3 * (size_t)Nk * (size_t)(n_or1(c))));
    CUDA_TRY(c, cudaMalloc(&D.P, sizeof(double) * 3 * (size_t)Qk * (size_t)(n_or1(c))));
  }
  CUDA_TRY(c, cudaMalloc(&D.AB, sizeof(double) * 8 * (size_t)NFk * (size_t)(c->n_tet > 0 ? c->n_tet : 1)));
  if (c->sparse_curl) {   // ĉ scratch of the streamed curl sweeps, rows of whole 16-mode chunks
    D.ldc = (c->p * (c->p + 1) * (c->p + 2) / 6 + 15) / 16 * 16;
    CUDA_TRY(c, cudaMalloc(&D.Cc, sizeof(double) * 3 * (size_t)D.ldc * (size_t)c->n_tet));
  }
  if (!(std::getenv("DGM_TILE_ORDER") && std::atoi(std::getenv("DGM_TILE_ORDER")) == 0))   // 0: static order
  {
    CUDA_TRY(c, cudaMalloc(&D.tile_ctr, 64));
    CUDA_TRY(c, cudaMemset(D.tile_ctr, 0, 64));   // then self-resetting (gemm_kernel)
  }
  return DGM_OK;
}

void free_ctx(dgm_ctx *c) {
  if (!c) return;
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  for (int i = 0; i < 2; ++i)
    if (c->gev[i]) cudaEventDestroy(c->gev[i]);
  cudaFree(c->d_dense);
  cudaFree(c->dense.AB);
  cudaFree(c->dense.tile_ctr);
  cudaFree(c->dense.Cc);
  for (void *q : {(void *)c->dense.Bf, (void *)c->dense.Bb, (void *)c->dense.ktlf, (void *)c->dense.ktofff,
                  (void *)c->dense.ktlb, (void *)c->dense.ktoffb, (void *)c->dense.SWe, (void *)c->dense.SWm,
                  (void *)c->dense.AC, (void *)c->dense.P, (void *)c->dense.KE, (void *)c->dense.KH,
                  (void *)c->dense.sf_tab, (void *)c->dense.sf_modes, (void *)c->dense.sf_pairs})
    cudaFree(q);
  cudaFree(c->d_stream);
  cudaFree(c->d_geo);
  cudaFree(c->d_nbr);
  cudaFree(c->d_nbrf);
  cudaFree(c->d_fmet);
  cudaFree(c->d_blob);
  for (int i = 0; i < 4; ++i) cudaFree(c->d_tr[i]);
  cudaFree(c->d_partial);
  cudaFree(c->d_E);
  cudaFree(c->d_H);
  for (int i = 0; i < 3; ++i) cudaFree(c->d_pw[i]);
  cudaFree(c->d_fid);
  cudaFree(c->d_fside);
  cudaFree(c->d_sign);
  cudaFree(c->d_fgeo);
  cudaFree(c->d_fnorms);
  if (c->side) cudaStreamDestroy(c->side);
  for (int i = 0; i < 4; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  delete c;
}

dgm_status create_impl(dgm_ctx *c, const dgm_mesh *m, int order, const double *eps, const double *mu,
                       const dgm_opts *opts) {
  if (!m || !m->xyz || !m->tet || m->n_vert <= 0 || m->n_tet <= 0 || !eps || !mu)
    return dgm::set_err(c, DGM_EINVAL, "null mesh/eps/mu pointer or empty mesh");
  if (order < 1 || order > DGM_PMAX)
    return dgm::set_err(c, DGM_EORDER, "order " + std::to_string(order) + " outside 1.." + std::to_string(DGM_PMAX));
  if (m->n_tet > (int64_t)INT32_MAX / 4) return dgm::set_err(c, DGM_EINVAL, "too many tets");
  dgm_opts o = opts ? *opts : dgm_opts{DGM_FLUX_CENTRAL, 0, 0, 0.0, DGM_ENGINE_AUTO, 0, 0, nullptr};
  if (o.engine < DGM_ENGINE_AUTO || o.engine > DGM_ENGINE_HYBRID) return dgm::set_err(c, DGM_EINVAL, "unknown engine");
  if (o.flux != DGM_FLUX_CENTRAL && o.flux != DGM_FLUX_UPWIND && o.flux != DGM_FLUX_STABILIZED)
    return dgm::set_err(c, DGM_EINVAL, "unknown flux");
  const int p = order;
  const int64_t n = m->n_tet;
  c->p = p;
  c->N = (p + 1) * (p + 2) * (p + 3) / 6;
  c->NF = (p + 1) * (p + 2) / 2;
  c->LD = (c->N + 3) & ~3;
  c->n_tet = n;
  c->flux = o.flux;
  // engine: explicit option, else DGM_ENGINE, else by order (measured): the
  // sparse recurrence kernels for p <= 5, dense DMMA contractions at p = 6, and from p = 7
  // the hybrid (the curl by the streamed recurrence sweeps, DMMA lift and traces; with the
  // constant-table sweeps C4 5.79 vs 5.84 ms and C5 46.9 vs 48.3 ms per step against dense)
  int kind = o.engine;
  if (kind == DGM_ENGINE_AUTO) {
    kind = p >= dgm::kHybridAuto ? DGM_ENGINE_HYBRID : p >= 6 ? DGM_ENGINE_DENSE : DGM_ENGINE_SPARSE;
    if (const char *v = std::getenv("DGM_ENGINE"))
      kind = std::strcmp(v, "dense") == 0 ? DGM_ENGINE_DENSE
             : std::strcmp(v, "hybrid") == 0 && p >= dgm::kCurlPmin ? DGM_ENGINE_HYBRID
                                                                     : DGM_ENGINE_SPARSE;
  }
  if (kind == DGM_ENGINE_HYBRID && (p < dgm::kCurlPmin || p > dgm::kCurlPmax))
    return dgm::set_err(c, DGM_EINVAL, "the hybrid engine covers orders 4..10");
  c->engine = kind == DGM_ENGINE_SPARSE ? 0 : 1;
  c->sparse_curl = kind == DGM_ENGINE_HYBRID ? 1 : 0;
  // mixed orders E ∈ P^p, H ∈ P^{p-1}: dense engine, central/upwind
  if (o.mixed_order) {
    if (p < 2) return dgm::set_err(c, DGM_EORDER, "mixed orders need order >= 2");
    if (o.flux == DGM_FLUX_STABILIZED) return dgm::set_err(c, DGM_EINVAL, "mixed orders: central or upwind flux only");
    if (o.engine == DGM_ENGINE_SPARSE || o.engine == DGM_ENGINE_HYBRID)
      return dgm::set_err(c, DGM_EINVAL, "mixed orders need the dense engine");
    c->engine = 1;
    c->sparse_curl = 0;   // the generated sweeps are equal-order
    c->mixed = 1;
  }
  c->NH = c->mixed ? p * (p + 1) * (p + 2) / 6 : c->N;
  // materials at the quadrature points (reverse numerical integration)
  if (o.material_points) {
    if (o.flux != DGM_FLUX_CENTRAL) return dgm::set_err(c, DGM_EINVAL, "material_points: central flux only");
    if (o.mixed_order) return dgm::set_err(c, DGM_EINVAL, "material_points: not with mixed orders");
    if (o.engine == DGM_ENGINE_SPARSE) return dgm::set_err(c, DGM_EINVAL, "material_points need the dense engine");
    c->engine = 1;
    c->matq = 1;
    std::vector<double> xi, w;
    tet_quadrature(p, xi, w);
    const int64_t Q = (int64_t)w.size();
    c->Q = (int)Q;
    c->Qk = (int)((Q + 15) / 16 * 16);
    c->h_swe.assign((size_t)n * c->Qk, 0.0);
    c->h_swm.assign((size_t)n * c->Qk, 0.0);
    for (int64_t t = 0; t < n; ++t)
      for (int64_t i = 0; i < Q; ++i) {
        const double e = eps[t * Q + i], u = mu[t * Q + i];
        if (!(e > 0) || !(u > 0) || !std::isfinite(e) || !std::isfinite(u))
          return dgm::set_err(c, DGM_EINVAL, "tet " + std::to_string(t) + ": point eps/mu must be positive");
        c->h_swe[(size_t)t * c->Qk + i] = w[i] / e;   // quadrature weight / material
        c->h_swm[(size_t)t * c->Qk + i] = w[i] / u;
      }
  }
  // curved (quadratic) elements: the same point pipeline with a 3x3 mix per point
  if (o.edge_nodes) {
    if (o.flux != DGM_FLUX_CENTRAL) return dgm::set_err(c, DGM_EINVAL, "curved elements: central flux only");
    if (o.mixed_order) return dgm::set_err(c, DGM_EINVAL, "curved elements: not with mixed orders");
    if (o.engine == DGM_ENGINE_SPARSE) return dgm::set_err(c, DGM_EINVAL, "curved elements need the dense engine");
    c->engine = 1;
    c->matq = 1;
    c->curved = 1;
    if (!o.material_points) {
      std::vector<double> xi, w;
      tet_quadrature(p, xi, w);
      c->Q = (int)w.size();
      c->Qk = (c->Q + 15) / 16 * 16;
    }
  }
  auto rep = [&](int32_t v) -> int64_t { return m->rep ? (int64_t)m->rep[v] : (int64_t)v; };

  // ---- validate vertex ids and canonical (ascending-rep) order
  for (int64_t t = 0; t < n; ++t) {
    for (int k = 0; k < 4; ++k) {
      int32_t v = m->tet[4 * t + k];
      if (v < 0 || v >= m->n_vert)
        return dgm::set_err(c, DGM_EMESH, "tet " + std::to_string(t) + ": vertex id out of range");
    }
    for (int k = 0; k < 3; ++k)
      if (!(rep(m->tet[4 * t + k]) < rep(m->tet[4 * t + k + 1])))
        return dgm::set_err(c, DGM_EMESH, "tet " + std::to_string(t) + ": vertices not strictly ascending by rep");
  }
  // ---- materials
  std::vector<double> ev(n), mv(n);
  for (int64_t t = 0; t < n; ++t) {
    ev[t] = c->matq ? 1.0 : o.eps_per_elem ? eps[t] : eps[0];   // point materials: applied in the inverse mass
    mv[t] = c->matq ? 1.0 : o.mu_per_elem ? mu[t] : mu[0];
    if (!(ev[t] > 0) || !(mv[t] > 0) || !std::isfinite(ev[t]) || !std::isfinite(mv[t]))
      return dgm::set_err(c, DGM_EINVAL, "tet " + std::to_string(t) + ": eps/mu must be positive");
  }
  // ---- geometry: F = [X1-X0, X2-X0, X3-X0]
  std::vector<Geo> geo(n);
  std::vector<double> fmet(o.flux == DGM_FLUX_UPWIND ? n * 12 : 0);
  std::vector<int8_t> sgn(n);
  for (int64_t t = 0; t < n; ++t) {
    double X[4][3];
    for (int k = 0; k < 4; ++k)
      for (int i = 0; i < 3; ++i) X[k][i] = m->xyz[3 * (int64_t)m->tet[4 * t + k] + i];
    double F[3][3];
    double L = 0;
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) F[i][j] = X[j + 1][i] - X[0][i];
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        double d2 = 0;
        for (int i = 0; i < 3; ++i) d2 += (X[a][i] - X[b][i]) * (X[a][i] - X[b][i]);
        L = std::max(L, std::sqrt(d2));
      }
    double det = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                 F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
    if (!(std::fabs(det) > 1e-12 * L * L * L))
      return dgm::set_err(c, DGM_EMESH, "tet " + std::to_string(t) + ": degenerate (|det F| too small)");
    double FtF[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int i = 0; i < 3; ++i) s += F[i][a] * F[i][b];
        FtF[a][b] = s;
      }
    Geo &g = geo[t];
    g.g[0] = FtF[0][0] / det;
    g.g[1] = FtF[0][1] / det;
    g.g[2] = FtF[0][2] / det;
    g.g[3] = FtF[1][1] / det;
    g.g[4] = FtF[1][2] / det;
    g.g[5] = FtF[2][2] / det;
    g.detF = det;
    g.inv_eps = 1.0 / ev[t];
    g.inv_mu = 1.0 / mv[t];
    g.Z = std::sqrt(mv[t] / ev[t]);
    sgn[t] = det > 0 ? 1 : -1;
    if (o.flux == DGM_FLUX_UPWIND) {
      for (int f = 0; f < 4; ++f) {
        const int *fv = kFaceVerts[f];
        double t1[3], t2[3];
        for (int i = 0; i < 3; ++i) {
          t1[i] = X[fv[1]][i] - X[fv[0]][i];
          t2[i] = X[fv[2]][i] - X[fv[0]][i];
        }
        double g11 = t1[0] * t1[0] + t1[1] * t1[1] + t1[2] * t1[2];
        double g12 = t1[0] * t2[0] + t1[1] * t2[1] + t1[2] * t2[2];
        double g22 = t2[0] * t2[0] + t2[1] * t2[1] + t2[2] * t2[2];
        double cx = t1[1] * t2[2] - t1[2] * t2[1], cy = t1[2] * t2[0] - t1[0] * t2[2], cz = t1[0] * t2[1] - t1[1] * t2[0];
        double area = std::sqrt(cx * cx + cy * cy + cz * cz);
        // M = |t1×t2| g^{-1},  det g = |t1×t2|²  (upwind tangential mass, reading G2)
        fmet[12 * t + 3 * f + 0] = g22 / area;
        fmet[12 * t + 3 * f + 1] = -g12 / area;
        fmet[12 * t + 3 * f + 2] = g11 / area;
      }
    }
  }
  // ---- curved elements: per quadrature point ξ_i the Jacobian F(ξ_i) of the quadratic
  // map and the point factor of the approximate inverse mass:
  //   K_i = ŵ_i F(ξ_i)ᵀF(ξ_i) / (m(x_i) det F(ξ_i))   (6 entries, symmetric)
  // the affine case gives K_i = ŵ_i G'/m, i.e. the flat path's G' and ŵ_i/m
  if (c->curved) {
    std::vector<double> xi, w;
    tet_quadrature(p, xi, w);
    const int Q = c->Q, Qk = c->Qk;
    c->h_ke.assign((size_t)n * Qk * 6, 0.0);
    c->h_kh.assign((size_t)n * Qk * 6, 0.0);
    static const int E[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    static const double GL[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};   // ∇λ_a
    for (int64_t t = 0; t < n; ++t) {
      double X[10][3];   // vertices, then edge nodes
      double L = 0;
      for (int k = 0; k < 4; ++k)
        for (int i = 0; i < 3; ++i) X[k][i] = m->xyz[3 * (int64_t)m->tet[4 * t + k] + i];
      for (int e = 0; e < 6; ++e)
        for (int i = 0; i < 3; ++i) {
          X[4 + e][i] = o.edge_nodes[(t * 6 + e) * 3 + i];
          if (!std::isfinite(X[4 + e][i]))
            return dgm::set_err(c, DGM_EINVAL, "tet " + std::to_string(t) + ": non-finite edge node");
        }
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b) {
          double d2 = 0;
          for (int i = 0; i < 3; ++i) d2 += (X[a][i] - X[b][i]) * (X[a][i] - X[b][i]);
          L = std::max(L, std::sqrt(d2));
        }
      for (int q = 0; q < Q; ++q) {
        const double *x = &xi[3 * q];
        const double lam[4] = {1.0 - x[0] - x[1] - x[2], x[0], x[1], x[2]};
        double F[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};   // F[i][j] = ∂Φ_i/∂ξ_j
        for (int j = 0; j < 3; ++j) {
          for (int a = 0; a < 4; ++a) {
            const double d = (4.0 * lam[a] - 1.0) * GL[a][j];
            for (int i = 0; i < 3; ++i) F[i][j] += d * X[a][i];
          }
          for (int e = 0; e < 6; ++e) {
            const int a = E[e][0], b = E[e][1];
            const double d = 4.0 * (GL[a][j] * lam[b] + lam[a] * GL[b][j]);
            for (int i = 0; i < 3; ++i) F[i][j] += d * X[4 + e][i];
          }
        }
        const double det = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
                           F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                           F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
        if (!(std::fabs(det) > 1e-12 * L * L * L) || (det > 0) != (sgn[t] > 0))
          return dgm::set_err(c, DGM_EMESH, "tet " + std::to_string(t) + ": curved map folds (det F changes sign)");
        double G[6];
        const int ij[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
        for (int k = 0; k < 6; ++k) {
          double sum = 0;
          for (int i = 0; i < 3; ++i) sum += F[i][ij[k][0]] * F[i][ij[k][1]];
          G[k] = sum / det;
        }
        const double me = o.material_points ? eps[t * Q + q] : o.eps_per_elem ? eps[t] : eps[0];
        const double mu_ = o.material_points ? mu[t * Q + q] : o.mu_per_elem ? mu[t] : mu[0];
        if (!(me > 0) || !(mu_ > 0) || !std::isfinite(me) || !std::isfinite(mu_))
          return dgm::set_err(c, DGM_EINVAL, "tet " + std::to_string(t) + ": eps/mu must be positive");
        for (int k = 0; k < 6; ++k) {
          c->h_ke[((size_t)t * Qk + q) * 6 + k] = w[q] * G[k] / me;
          c->h_kh[((size_t)t * Qk + q) * 6 + k] = w[q] * G[k] / mu_;
        }
      }
    }
  }
  // ---- face matching: sort representative triples (deterministic)
  std::vector<FaceRec> faces;
  try {
    faces.resize((size_t)n * 4);
  } catch (const std::bad_alloc &) {
    return dgm::set_err(c, DGM_ENOMEM, "host allocation for faces");
  }
  for (int64_t t = 0; t < n; ++t)
    for (int f = 0; f < 4; ++f) {
      FaceRec &r = faces[4 * t + f];
      for (int k = 0; k < 3; ++k) r.r[k] = (int32_t)rep(m->tet[4 * t + kFaceVerts[f][k]]);
      r.tet = (int32_t)t;
      r.f = (int8_t)f;
    }
  std::sort(faces.begin(), faces.end(), [](const FaceRec &a, const FaceRec &b) {
    if (a.r[0] != b.r[0]) return a.r[0] < b.r[0];
    if (a.r[1] != b.r[1]) return a.r[1] < b.r[1];
    if (a.r[2] != b.r[2]) return a.r[2] < b.r[2];
    if (a.tet != b.tet) return a.tet < b.tet;
    return a.f < b.f;
  });
  c->nbr.assign(n * 4, -1);
  c->nbrf.assign(n * 4, -1);
  c->bc.assign(n * 4, 1);
  c->sign.assign(n * 4, 0);
  for (size_t i = 0; i < faces.size();) {
    size_t j = i + 1;
    while (j < faces.size() && faces[j].r[0] == faces[i].r[0] && faces[j].r[1] == faces[i].r[1] &&
           faces[j].r[2] == faces[i].r[2])
      ++j;
    if (j - i > 2)
      return dgm::set_err(c, DGM_EMESH, "face of tet " + std::to_string(faces[i].tet) + " shared by more than two tets");
    if (j - i == 2) {
      const FaceRec &a = faces[i], &b = faces[i + 1];
      c->nbr[4 * a.tet + a.f] = b.tet;
      c->nbrf[4 * a.tet + a.f] = b.f;
      c->nbr[4 * b.tet + b.f] = a.tet;
      c->nbrf[4 * b.tet + b.f] = a.f;
      c->bc[4 * a.tet + a.f] = 0;
      c->bc[4 * b.tet + b.f] = 0;
    }
    i = j;
  }
  for (int64_t t = 0; t < n; ++t)
    for (int f = 0; f < 4; ++f) c->sign[4 * t + f] = (int8_t)((f % 2 == 0 ? 1 : -1) * sgn[t]);
  // curved elements: a face shared by two tets through the same three vertices must have
  // the same three edge nodes on both sides (conforming curved faces; periodic pairs
  // are the caller's responsibility)
  if (c->curved) {
    auto edge_of = [](int a, int b) { return a == 0 ? b - 1 : (a == 1 ? 2 + b - 1 : 5); };   // a < b
    for (int64_t t = 0; t < n; ++t)
      for (int f = 0; f < 4; ++f) {
        const int32_t s2 = c->nbr[4 * t + f];
        if (s2 < 0 || s2 < t) continue;
        const int g = c->nbrf[4 * t + f];
        const int *fa = kFaceVerts[f], *fb = kFaceVerts[g];
        bool same = true;
        for (int k = 0; k < 3; ++k) same &= m->tet[4 * t + fa[k]] == m->tet[4 * (int64_t)s2 + fb[k]];
        if (!same) continue;   // periodic pair
        for (int u = 0; u < 3; ++u)
          for (int v = u + 1; v < 3; ++v) {
            const double *pa = &o.edge_nodes[(t * 6 + edge_of(fa[u], fa[v])) * 3];
            const double *pb = &o.edge_nodes[((int64_t)s2 * 6 + edge_of(fb[u], fb[v])) * 3];
            if (pa[0] != pb[0] || pa[1] != pb[1] || pa[2] != pb[2])
              return dgm::set_err(c, DGM_EMESH, "tets " + std::to_string(t) + ", " + std::to_string(s2) +
                                                    ": shared face with different edge nodes");
          }
      }
  }

  // ---- stabilised central flux: face numbering and face geometry
  if (o.flux == DGM_FLUX_STABILIZED) {
    c->alpha = (o.alpha0 > 0 ? o.alpha0 : 1.0) * p * p;
    c->fid.assign(n * 4, -1);
    c->fside.clear();
    for (int64_t t = 0; t < n; ++t)
      for (int f = 0; f < 4; ++f) {
        const int32_t nb = c->nbr[4 * t + f];
        if (nb < 0 || t < nb) {
          c->fid[4 * t + f] = (int32_t)(c->fside.size() / 2);
          c->fside.push_back((int32_t)(4 * t + f));
          c->fside.push_back(nb < 0 ? -1 : 4 * nb + c->nbrf[4 * t + f]);
        }
      }
    for (int64_t t = 0; t < n; ++t)
      for (int f = 0; f < 4; ++f)
        if (c->fid[4 * t + f] < 0) c->fid[4 * t + f] = c->fid[4 * c->nbr[4 * t + f] + c->nbrf[4 * t + f]];
    c->n_faces = (int64_t)c->fside.size() / 2;
    c->fgeo.assign(c->n_faces * 8, 0.0);
    for (int64_t k = 0; k < c->n_faces; ++k) {
      const int64_t t = c->fside[2 * k] / 4;
      const int f = c->fside[2 * k] % 4;
      const int *fv = kFaceVerts[f];
      double X[3][3];
      for (int q = 0; q < 3; ++q)
        for (int i = 0; i < 3; ++i) X[q][i] = m->xyz[3 * (int64_t)m->tet[4 * t + fv[q]] + i];
      double t1[3], t2[3];
      for (int i = 0; i < 3; ++i) {
        t1[i] = X[1][i] - X[0][i];
        t2[i] = X[2][i] - X[0][i];
      }
      const double g11 = t1[0] * t1[0] + t1[1] * t1[1] + t1[2] * t1[2];
      const double g12 = t1[0] * t2[0] + t1[1] * t2[1] + t1[2] * t2[2];
      const double g22 = t2[0] * t2[0] + t2[1] * t2[1] + t2[2] * t2[2];
      const double cx = t1[1] * t2[2] - t1[2] * t2[1], cy = t1[2] * t2[0] - t1[0] * t2[2],
                   cz = t1[0] * t2[1] - t1[1] * t2[0];
      const double area = std::sqrt(cx * cx + cy * cy + cz * cz);
      double *G = &c->fgeo[8 * k];
      G[0] = g11 / area;   // M^{-1} = g / |t1×t2|
      G[1] = g12 / area;
      G[2] = g22 / area;
      G[3] = c->alpha / std::sqrt(area);   // α / h_F: Ḣ^F factor (reading G17), h_F = sqrt(|t1×t2|) (G16)
      G[4] = g22 / area;   // M = |t1×t2| g^{-1}
      G[5] = -g12 / area;
      G[6] = g11 / area;
    }
  }

  c->h_geo.swap(geo);
  c->h_fmet.swap(fmet);
  return DGM_OK;
}

dgm_status upload_impl(dgm_ctx *c) {
  const int64_t n = c->n_tet;
  const int p = c->p;
  int dev = 0;
  CUDA_TRY(c, cudaGetDevice(&dev));
  CUDA_TRY(c, cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev));
  if (const char *v = std::getenv("DGM_GRAPHS")) c->use_graphs = std::atoi(v) != 0;
  CUDA_TRY(c, cudaMalloc(&c->d_geo, sizeof(Geo) * n));
  CUDA_TRY(c, cudaMemcpy(c->d_geo, c->h_geo.data(), sizeof(Geo) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMalloc(&c->d_nbr, 4 * sizeof(int32_t) * n));
  CUDA_TRY(c, cudaMemcpy(c->d_nbr, c->nbr.data(), 4 * sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMalloc(&c->d_nbrf, 4 * n));
  CUDA_TRY(c, cudaMemcpy(c->d_nbrf, c->nbrf.data(), 4 * n, cudaMemcpyHostToDevice));
  if (c->flux == DGM_FLUX_UPWIND) {
    CUDA_TRY(c, cudaMalloc(&c->d_fmet, sizeof(double) * 12 * n));
    CUDA_TRY(c, cudaMemcpy(c->d_fmet, c->h_fmet.data(), sizeof(double) * 12 * n, cudaMemcpyHostToDevice));
  }
  if (c->flux == DGM_FLUX_STABILIZED) {
    CUDA_TRY(c, cudaMalloc(&c->d_fid, 4 * sizeof(int32_t) * n));
    CUDA_TRY(c, cudaMemcpy(c->d_fid, c->fid.data(), 4 * sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMalloc(&c->d_fside, 2 * sizeof(int32_t) * c->n_faces));
    CUDA_TRY(c, cudaMemcpy(c->d_fside, c->fside.data(), 2 * sizeof(int32_t) * c->n_faces, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMalloc(&c->d_sign, 4 * n));
    CUDA_TRY(c, cudaMemcpy(c->d_sign, c->sign.data(), 4 * n, cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMalloc(&c->d_fgeo, 8 * sizeof(double) * c->n_faces));
    CUDA_TRY(c, cudaMemcpy(c->d_fgeo, c->fgeo.data(), 8 * sizeof(double) * c->n_faces, cudaMemcpyHostToDevice));
    std::vector<double> fn(c->NF);
    for (int d = 0, q = 0; d <= p; ++d)
      for (int mm = 0; mm <= d; ++mm, ++q) fn[q] = 1.0 / ((2.0 * mm + 1) * (2.0 * d + 2));   // ‖ψ_mn‖², n = d-m
    CUDA_TRY(c, cudaMalloc(&c->d_fnorms, sizeof(double) * c->NF));
    CUDA_TRY(c, cudaMemcpy(c->d_fnorms, fn.data(), sizeof(double) * c->NF, cudaMemcpyHostToDevice));
  }
  // trace buffers TE0, TE1, TH0, TH1 (the second of each only for upwind); the lane
  // path interleaves groups of 16 elements, so round up, plus 16 spare elements that
  // absorb the writes of unused slots of a partial last group
  for (int i = 0; i < 4; ++i) {
    if ((i == 1 || i == 3) && c->flux != DGM_FLUX_UPWIND) continue;
    CUDA_TRY(c, cudaMalloc(&c->d_tr[i], sizeof(double) * ((n + 15) / 16 * 16 + 16) * 8 * c->NF));
  }
  const HostProgSet &hs = kHostProgs[p - 1];
  size_t bytes = prog_bytes(hs.curl) + 256 + (size_t)c->N * 8;
  for (int f = 0; f < 4; ++f)
    bytes += prog_bytes(hs.strace[f].prog) + prog_bytes(hs.slift[f].prog) + 2 * (((size_t)c->N * 2 + 255) & ~size_t(255));
  std::vector<char> buf(bytes, 0);
  CUDA_TRY(c, cudaMalloc(&c->d_blob, bytes));
  size_t off = 0;
  char *base = (char *)c->d_blob;
  c->progs.curl = stage_prog(hs.curl, buf, off, base);
  auto stage_sprog = [&](const dgm::HostSProg &h, int nout) {
    dgm::DevSProg d;
    d.prog = stage_prog(h.prog, buf, off, base);
    d.n_in = h.n_in;
    d.n_scr = h.n_scr;
    std::memcpy(buf.data() + off, h.out, nout * 2);
    d.out = (const uint16_t *)(base + off);
    off += ((size_t)nout * 2 + 255) & ~size_t(255);
    return d;
  };
  for (int f = 0; f < 4; ++f) {
    c->progs.strace[f] = stage_sprog(hs.strace[f], c->NF);
    c->progs.slift[f] = stage_sprog(hs.slift[f], c->N);
  }
  std::memcpy(buf.data() + off, hs.norms, c->N * 8);
  c->progs.norms = (const double *)(base + off);
  off += ((size_t)c->N * 8 + 255) & ~size_t(255);
  CUDA_TRY(c, cudaMemcpy(c->d_blob, buf.data(), bytes, cudaMemcpyHostToDevice));
  if (c->engine == 1) {
    dgm_status r = dense_build(c, hs);
    if (r != DGM_OK) return r;
  }
  if (p > dgm::kLanePmax) {
    const char *v = std::getenv("DGM_ST_CHUNK");
    const size_t cap = v && *v ? (size_t)std::atol(v) : 16384;
    dgm_status r = build_stream(c, hs, cap);
    if (r != DGM_OK) return r;
  }
  return DGM_OK;
}

}  // namespace

extern "C" {

dgm_status dgm_create(const dgm_mesh *mesh, int order, const double *eps, const double *mu, const dgm_opts *opts,
                      dgm_ctx **out) {
  if (!out) return DGM_EINVAL;
  *out = nullptr;
  dgm_ctx *c = new (std::nothrow) dgm_ctx();
  if (!c) return DGM_ENOMEM;
  dgm_status s = create_impl(c, mesh, order, eps, mu, opts);
  if (s == DGM_OK) s = upload_impl(c);
  if (s != DGM_OK) {
    g_create_err = c->err;   // reachable as dgm_last_error(NULL)
    free_ctx(c);
    return s;
  }
  *out = c;
  return DGM_OK;
}

dgm_status dgm_match_faces_host(const dgm_mesh *mesh, int32_t *nbr, int8_t *nbr_face, int8_t *sign, int8_t *bc) {
  dgm_ctx tmp;
  double one = 1.0;
  dgm_status s = create_impl(&tmp, mesh, 1, &one, &one, nullptr);
  if (s != DGM_OK) {
    g_create_err = tmp.err;
    return s;
  }
  return dgm_tables(&tmp, nbr, nbr_face, sign, bc);
}

dgm_status dgm_layout(const dgm_ctx *c, int64_t *n_modes, int64_t *ld, int64_t *n_tet) {
  if (!c) return DGM_EINVAL;
  if (n_modes) *n_modes = c->N;
  if (ld) *ld = c->LD;
  if (n_tet) *n_tet = c->n_tet;
  return DGM_OK;
}

dgm_status dgm_apply_curl(dgm_ctx *c, const double *E, const double *H, double *dE, double *dH, void *stream) {
  if (!c || !E || !H) return dgm::set_err(c, DGM_EINVAL, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  c->launches = 0;
  dgm_status s = DGM_OK;
  if (dE) s = dgm::launch_tb_stage(c, dgm::STAGE_E, H, nullptr, dE, 0.0, 1, 0, dgm::OUT_WRITE, nullptr, nullptr, nullptr, st);
  if (s == DGM_OK && dH)
    s = dgm::launch_tb_stage(c, dgm::STAGE_H, E, nullptr, dH, 0.0, 1, 0, dgm::OUT_WRITE, nullptr, nullptr, nullptr, st);
  return s;
}

dgm_status dgm_apply_flux(dgm_ctx *c, const double *E, const double *H, double *dE, double *dH, int accumulate,
                          void *stream) {
  if (!c || !E || !H) return dgm::set_err(c, DGM_EINVAL, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  int om = accumulate ? dgm::OUT_ACCUM : dgm::OUT_WRITE;
  c->launches = 0;
  // traces of both fields, then the face parts: the E equation reads H's traces
  // (and, upwind, E's own), the H equation the other way round
  double *TE = c->d_tr[0], *TH = c->d_tr[2];
  c->tr_valid = false;   // the buffers now hold the traces of these E, H
  dgm_status s = dgm::launch_tb_traces(c, E, TE, st, 0);
  if (s == DGM_OK) s = dgm::launch_tb_traces(c, H, TH, st, 1);
  if (s == DGM_OK && dE) s = dgm::launch_tb_stage(c, dgm::STAGE_E, H, nullptr, dE, 0.0, 0, 1, om, TH, TE, nullptr, st);
  if (s == DGM_OK && dH) s = dgm::launch_tb_stage(c, dgm::STAGE_H, E, nullptr, dH, 0.0, 0, 1, om, TE, TH, nullptr, st);
  return s;
}

dgm_status dgm_step(dgm_ctx *c, double *E, double *H, double dt, int64_t nsteps, void *stream) {
  return dgm_step_ex(c, E, H, dt, nsteps, 0, stream);
}

namespace {
// The step sequence of dgm_step_ex.  If h_done is given it is recorded on the
// stream right after the last H stage (H is final from then on).  If
// before_entry is given the stream waits on it after the entry traces of E.
dgm_status run_steps(dgm_ctx *c, double *E, double *H, double dt, int64_t nsteps, int flags, cudaStream_t st,
                     cudaEvent_t before_h, cudaEvent_t h_done, double *HF = nullptr) {
  if (c->flux == DGM_FLUX_STABILIZED && !HF)
    return dgm::set_err(c, DGM_EINVAL, "stabilised contexts step through dgm_step_sc (the face unknowns H^F)");
  const bool up = c->flux == DGM_FLUX_UPWIND;
  int ce = 0, ch = 0;
  dgm_status r = DGM_OK;
  if ((flags & DGM_STEP_CONTINUE) && c->tr_valid && c->tr_E == E && c->tr_H == H) {
    ce = c->tr_ce;
    ch = c->tr_ch;
    if (before_h) cudaStreamWaitEvent(st, before_h, 0);
  } else {
    r = dgm::launch_tb_traces(c, E, c->d_tr[0], st, 0);
    if (before_h) cudaStreamWaitEvent(st, before_h, 0);   // H has arrived
    if (r == DGM_OK && up) r = dgm::launch_tb_traces(c, H, c->d_tr[2], st, 1);
  }
  c->tr_valid = false;
  // one symplectic-Euler step on stream ss (ce, ch: current trace-buffer parities)
  auto one_step = [&](cudaStream_t ss, bool last) -> dgm_status {
    double *TE = c->d_tr[ce], *THr = c->d_tr[2 + ch], *THw = c->d_tr[2 + (up ? 1 - ch : ch)];
    dgm_status q = dgm::launch_tb_stage(c, dgm::STAGE_H, E, H, nullptr, dt, 1, 1, dgm::OUT_UPDATE, TE, THr, THw, ss);
    if (up) ch = 1 - ch;
    if (q != DGM_OK) return q;
    // stabilised flux: H^F += dt Ḣ^F(E^n) from E's traces (before the E stage overwrites them)
    if (HF && (q = dgm::launch_hf(c, TE, HF, nullptr, dt, ss)) != DGM_OK) return q;
    if (h_done && last) cudaEventRecord(h_done, ss);
    double *TH = c->d_tr[2 + ch], *TEw = c->d_tr[up ? 1 - ce : ce];
    c->cur_HF = HF;
    q = dgm::launch_tb_stage(c, dgm::STAGE_E, H, E, nullptr, dt, 1, 1, dgm::OUT_UPDATE, TH, c->d_tr[ce], TEw, ss);
    c->cur_HF = nullptr;
    if (up) ce = 1 - ce;
    return q;
  };
  int64_t s = 0;
  // Long runs: replay a captured CUDA graph of kGraphSteps steps (an even count, so
  // the upwind trace-buffer parities return to where they started and one graph
  // serves every chunk).  Small meshes are launch-bound; the graph removes the
  // per-kernel launch cost.  Same kernels, same order: bit-identical results.
  constexpr int64_t kGraphSteps = 32;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);   // the caller may be capturing us into its own graph
  const bool graphs = c->use_graphs && !h_done && nsteps >= 2 * kGraphSteps && r == DGM_OK &&
                      cap == cudaStreamCaptureStatusNone;
  if (graphs) {
    const GraphKey key{E, H, HF, dt, ce, ch};
    if (!c->gexec || !(c->gkey == key)) {
      if (c->gexec) cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
      if (!c->gstream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking));
      const int ce0 = ce, ch0 = ch;
      const int64_t l0 = c->launches;
      cudaGraph_t g = nullptr;
      CUDA_TRY(c, cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeThreadLocal));
      for (int64_t k = 0; k < kGraphSteps && r == DGM_OK; ++k) r = one_step(c->gstream, false);
      cudaError_t ec = cudaStreamEndCapture(c->gstream, &g);
      if (r != DGM_OK) {
        if (g) cudaGraphDestroy(g);
        return r;
      }
      if (ec != cudaSuccess) return dgm::set_err(c, DGM_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
      ec = cudaGraphInstantiate(&c->gexec, g, 0);
      cudaGraphDestroy(g);
      if (ec != cudaSuccess) return dgm::set_err(c, DGM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ec));
      c->gkey = key;
      c->glaunches = c->launches - l0;
      c->launches = l0;
      ce = ce0;
      ch = ch0;
    }
    if (!c->gev[0]) {
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->gev[0], cudaEventDisableTiming));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->gev[1], cudaEventDisableTiming));
    }
    CUDA_TRY(c, cudaEventRecord(c->gev[0], st));
    CUDA_TRY(c, cudaStreamWaitEvent(c->gstream, c->gev[0], 0));
    for (; s + kGraphSteps <= nsteps; s += kGraphSteps) {
      CUDA_TRY(c, cudaGraphLaunch(c->gexec, c->gstream));
      c->launches += c->glaunches;
    }
    CUDA_TRY(c, cudaEventRecord(c->gev[1], c->gstream));
    CUDA_TRY(c, cudaStreamWaitEvent(st, c->gev[1], 0));
  }
  for (; s < nsteps && r == DGM_OK; ++s) r = one_step(st, s == nsteps - 1);
  if (r == DGM_OK) {
    c->tr_valid = true;
    c->tr_E = E;
    c->tr_H = H;
    c->tr_ce = ce;
    c->tr_ch = ch;
  }
  return r;
}
}  // namespace

dgm_status dgm_step_ex(dgm_ctx *c, double *E, double *H, double dt, int64_t nsteps, int flags, void *stream) {
  if (!c || !E || !H || nsteps < 0 || !std::isfinite(dt)) return dgm::set_err(c, DGM_EINVAL, "bad step arguments");
  c->launches = 0;
  if (nsteps == 0) return DGM_OK;
  // Each stage reads the traces of the field it does not update (own and
  // neighbours) from the buffer written by the stage that last updated that
  // field, and writes the traces of the field it updates.  They are recomputed
  // at entry so that resuming from saved (E, H) is exact.  Upwind also reads
  // the old traces of the updated field, so those buffers ping-pong.
  return run_steps(c, E, H, dt, nsteps, flags, (cudaStream_t)stream, nullptr, nullptr);
}

dgm_status dgm_step_host(dgm_ctx *c, double *Eh, double *Hh, double dt, int64_t nsteps, void *stream) {
  if (!c || !Eh || !Hh || nsteps < 0 || !std::isfinite(dt)) return dgm::set_err(c, DGM_EINVAL, "bad step arguments");
  if (c->flux == DGM_FLUX_STABILIZED)   // checked before any copy is enqueued
    return dgm::set_err(c, DGM_EINVAL, "stabilised contexts step through dgm_step_sc (the face unknowns H^F)");
  cudaStream_t st = (cudaStream_t)stream;
  size_t bytes = sizeof(double) * 3 * (size_t)c->n_tet * c->LD;
  if (!c->d_E) {
    CUDA_TRY(c, cudaMalloc(&c->d_E, bytes));
    CUDA_TRY(c, cudaMalloc(&c->d_H, bytes));
  }
  if (!c->side) {
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    for (int i = 0; i < 4; ++i) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  }
  c->launches = 0;
  if (nsteps == 0) return DGM_OK;
  // E in on the caller's stream (the entry traces of E start as soon as it lands),
  // H in on a side stream; H back out on the side stream as soon as the last H
  // stage is done, overlapping the last E stage; E back out last.
  CUDA_TRY(c, cudaEventRecord(c->ev[0], st));                 // caller's prior work
  CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev[0], 0));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_E, Eh, bytes, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_H, Hh, bytes, cudaMemcpyHostToDevice, c->side));
  CUDA_TRY(c, cudaEventRecord(c->ev[1], c->side));           // H has arrived
  c->tr_valid = false;   // fresh host data
  dgm_status s = run_steps(c, c->d_E, c->d_H, dt, nsteps, 0, st, c->ev[1], c->ev[2]);
  if (s != DGM_OK) {
    cudaStreamSynchronize(c->side);   // no copy outlives a failed call
    cudaStreamSynchronize(st);
    return s;
  }
  CUDA_TRY(c, cudaStreamWaitEvent(c->side, c->ev[2], 0));    // last H stage done
  CUDA_TRY(c, cudaMemcpyAsync(Hh, c->d_H, bytes, cudaMemcpyDeviceToHost, c->side));
  CUDA_TRY(c, cudaEventRecord(c->ev[3], c->side));
  CUDA_TRY(c, cudaMemcpyAsync(Eh, c->d_E, bytes, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev[3], 0));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  c->tr_valid = false;   // the caller owns the host copies now
  return DGM_OK;
}

dgm_status dgm_faces(const dgm_ctx *c, int64_t *n_faces, int32_t *face_id) {
  if (!c) return DGM_EINVAL;
  if (c->flux != DGM_FLUX_STABILIZED) return DGM_EINVAL;
  if (n_faces) *n_faces = c->n_faces;
  if (face_id) std::memcpy(face_id, c->fid.data(), sizeof(int32_t) * 4 * c->n_tet);
  return DGM_OK;
}

dgm_status dgm_step_sc(dgm_ctx *c, double *E, double *H, double *HF, double dt, int64_t nsteps, int flags,
                       void *stream) {
  if (!c || !E || !H || !HF || nsteps < 0 || !std::isfinite(dt)) return dgm::set_err(c, DGM_EINVAL, "bad step arguments");
  if (c->flux != DGM_FLUX_STABILIZED) return dgm::set_err(c, DGM_EINVAL, "context was not created with DGM_FLUX_STABILIZED");
  c->launches = 0;
  if (nsteps == 0) return DGM_OK;
  return run_steps(c, E, H, dt, nsteps, flags, (cudaStream_t)stream, nullptr, nullptr, HF);
}

dgm_status dgm_rhs_sc(dgm_ctx *c, const double *E, const double *H, const double *HF, double *dE, double *dH,
                      double *dHF, void *stream) {
  if (!c || !E || !H || !HF) return dgm::set_err(c, DGM_EINVAL, "null pointer");
  if (c->flux != DGM_FLUX_STABILIZED) return dgm::set_err(c, DGM_EINVAL, "context was not created with DGM_FLUX_STABILIZED");
  cudaStream_t st = (cudaStream_t)stream;
  c->launches = 0;
  c->tr_valid = false;
  double *TE = c->d_tr[0], *TH = c->d_tr[2];
  dgm_status s = dgm::launch_tb_traces(c, E, TE, st, 0);
  if (s == DGM_OK) s = dgm::launch_tb_traces(c, H, TH, st, 1);
  if (s == DGM_OK && dH) s = dgm::launch_tb_stage(c, dgm::STAGE_H, E, nullptr, dH, 0.0, 1, 1, dgm::OUT_WRITE, TE, TH, nullptr, st);
  if (s == DGM_OK && dHF) s = dgm::launch_hf(c, TE, nullptr, dHF, 0.0, st);
  if (s == DGM_OK && dE) {
    c->cur_HF = HF;
    s = dgm::launch_tb_stage(c, dgm::STAGE_E, H, nullptr, dE, 0.0, 1, 1, dgm::OUT_WRITE, TH, TE, nullptr, st);
    c->cur_HF = nullptr;
  }
  return s;
}

dgm_status dgm_energy_sc(dgm_ctx *c, const double *E, const double *H, const double *HF, double *out, void *stream) {
  if (!c || !E || !H || !HF || !out) return dgm::set_err(c, DGM_EINVAL, "null pointer");
  if (c->flux != DGM_FLUX_STABILIZED) return dgm::set_err(c, DGM_EINVAL, "context was not created with DGM_FLUX_STABILIZED");
  double w = 0.0, wf = 0.0;
  dgm_status s = dgm::launch_energy(c, E, H, &w, (cudaStream_t)stream);
  if (s == DGM_OK) s = dgm::launch_face_energy(c, HF, &wf, (cudaStream_t)stream);
  if (s == DGM_OK) *out = w + wf;
  return s;
}

dgm_status dgm_spectral_radius(dgm_ctx *c, int iters, uint64_t seed, double *rho_out, void *stream) {
  if (!c || !rho_out || iters < 1) return dgm::set_err(c, DGM_EINVAL, "bad spectral_radius arguments");
  if (c->matq) return dgm::set_err(c, DGM_EINVAL, "spectral_radius: not for material_points contexts");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * 3 * (size_t)c->n_tet * c->LD;
  for (int i = 0; i < 3; ++i)
    if (!c->d_pw[i]) {
      CUDA_TRY(c, cudaMalloc(&c->d_pw[i], bytes));
      CUDA_TRY(c, cudaMemsetAsync(c->d_pw[i], 0, bytes, st));
    }
  double *Hv = c->d_pw[0], *D = c->d_pw[1], *W = c->d_pw[2];
  c->tr_valid = false;   // the trace buffers are used as scratch here
  dgm_status r = dgm::launch_seed(c, Hv, seed, st);
  // zero field for the "other" argument (E = 0 for Ė(0, H); H = 0 for Ḣ(D, 0))
  double *Z = W;
  double rho = 0.0;
  for (int it = 0; it < iters && r == DGM_OK; ++it) {
    double nrm2 = 0.0;
    if ((r = dgm::launch_massdot(c, Hv, Hv, 1, &nrm2, st)) != DGM_OK) break;
    if (!(nrm2 > 0.0) || !std::isfinite(nrm2)) return dgm::set_err(c, DGM_EINVAL, "power iteration broke down");
    if ((r = dgm::launch_scale(c, Hv, Hv, 1.0 / std::sqrt(nrm2), st)) != DGM_OK) break;
    // D = Ė(0, H) = -Mε^{-1} Cᵀ H   (curl + face parts; upwind E-terms vanish for E = 0)
    CUDA_TRY(c, cudaMemsetAsync(Z, 0, bytes, st));
    if ((r = dgm::launch_tb_traces(c, Hv, c->d_tr[2], st, 1)) != DGM_OK) break;
    if ((r = dgm::launch_tb_traces(c, Z, c->d_tr[0], st, 0)) != DGM_OK) break;
    if ((r = dgm::launch_tb_stage(c, dgm::STAGE_E, Hv, nullptr, D, 0.0, 1, 1, dgm::OUT_WRITE, c->d_tr[2], c->d_tr[0],
                                  nullptr, st)) != DGM_OK)
      break;
    // W = Ḣ(D, 0) = Mμ^{-1} C D
    if ((r = dgm::launch_tb_traces(c, D, c->d_tr[0], st, 0)) != DGM_OK) break;
    if ((r = dgm::launch_tb_traces(c, Z, c->d_tr[2], st, 1)) != DGM_OK) break;
    if ((r = dgm::launch_tb_stage(c, dgm::STAGE_H, D, nullptr, W, 0.0, 1, 1, dgm::OUT_WRITE, c->d_tr[0], c->d_tr[2],
                                  nullptr, st)) != DGM_OK)
      break;
    // K H = -W;  Rayleigh quotient ρ = (H, Mμ K H) with ‖H‖_Mμ = 1
    double hw = 0.0;
    if ((r = dgm::launch_massdot(c, Hv, W, 1, &hw, st)) != DGM_OK) break;
    rho = -hw;
    if ((r = dgm::launch_scale(c, Hv, W, -1.0, st)) != DGM_OK) break;
  }
  if (r != DGM_OK) return r;
  *rho_out = rho;
  return DGM_OK;
}

dgm_status dgm_energy(dgm_ctx *c, const double *E, const double *H, double *out, void *stream) {
  if (!c || !E || !H || !out) return dgm::set_err(c, DGM_EINVAL, "null pointer");
  if (c->matq) return dgm::set_err(c, DGM_EINVAL, "dgm_energy: not for material_points contexts");
  return dgm::launch_energy(c, E, H, out, (cudaStream_t)stream);
}

dgm_status dgm_tables(const dgm_ctx *c, int32_t *nbr, int8_t *nbr_face, int8_t *sign, int8_t *bc) {
  if (!c) return DGM_EINVAL;
  size_t n = (size_t)c->n_tet * 4;
  if (nbr) std::memcpy(nbr, c->nbr.data(), n * 4);
  if (nbr_face) std::memcpy(nbr_face, c->nbrf.data(), n);
  if (sign) std::memcpy(sign, c->sign.data(), n);
  if (bc) std::memcpy(bc, c->bc.data(), n);
  return DGM_OK;
}

dgm_status dgm_quadrature_host(int order, int64_t *Q, double *xi, double *w) {
  if (order < 1 || order > DGM_PMAX || !Q) return DGM_EINVAL;
  std::vector<double> x, ww;
  tet_quadrature(order, x, ww);
  *Q = (int64_t)ww.size();
  if (xi) std::memcpy(xi, x.data(), x.size() * 8);
  if (w) std::memcpy(w, ww.data(), ww.size() * 8);
  return DGM_OK;
}

int dgm_engine(const dgm_ctx *c) {
  if (!c) return -1;
  return c->engine == 0 ? DGM_ENGINE_SPARSE : (c->sparse_curl ? DGM_ENGINE_HYBRID : DGM_ENGINE_DENSE);
}

int64_t dgm_last_launches(const dgm_ctx *c) { return c ? c->launches : 0; }

const char *dgm_last_error(const dgm_ctx *c) { return c ? c->err.c_str() : g_create_err.c_str(); }

void dgm_destroy(dgm_ctx *c) { free_ctx(c); }

}  // extern "C"
