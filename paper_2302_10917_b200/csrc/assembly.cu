// Device assembly of the 2-D HDG blocks.
//
// Replaces assemble_macro / assemble_face (mehdg/assembly.py:170-322) for a
// conforming structured macro mesh: one CTA per macro computes, from the
// reference-element tables (paper_2302_10917_b200/fem.py), the two sub-cell
// class tables of the red pattern (mass M, the gradient couplings K_x, K_y
// and, with SUPG, the streamline term S) and scatters them over the m^2
// sub-cells into the dense local block A ([q_x | q_y | u], 3Q x 3Q), then
// adds the boundary terms of the three faces to A, op.B and op.C and the
// Dirichlet trace elimination to R_u.  Contributions are added in the
// reference's order per entry; sub-cells and faces are processed one after the
// other with a CTA barrier in between (no atomics: deterministic).
// A second kernel forms the face blocks D = (sum over sides of a.n - tau) Mface.

#include <algorithm>
#include <cmath>

#include "mh_internal.h"

namespace mh {
namespace {

constexpr int kAsmThreads = 128;

struct AsmDev {
  mh_hdg2d_tables T;
  int64_t N;
  const double* verts;        // N x 3 x 2
  int S;                      // face slots per macro (3; up to 6 with hanging faces)
  const int8_t* slot_edge;    // N x S: local edge of the slot's face, -1 = empty slot
  const int8_t* slot_var;     // N x S: side variant (fem.SIDE_VARIANTS: t0, t1)
  const int32_t* slot_dir;    // N x S: row of ghat for a Dirichlet face, else -1
  const double* slot_len;     // N x S: face length
  const double* ghat;         // nD x t
  const double* fq;           // N x ncell x nq
  double* A;                  // N x nloc x nloc
  double* B;                  // N x nloc x nc   (op.B)
  double* C;                  // N x nc x nloc   (op.C)
  double* Ru;                 // N x nloc
};

struct Geo {
  double J[2][2];  // columns v1 - v0, v2 - v0
  double nrm[3][2];
  double len[3];
  double diam;
};

__device__ void geometry(const double* v, Geo& g) {
  const int ev[3][2] = {{1, 2}, {2, 0}, {0, 1}};  // EDGE_VERTS, mesh.py:68
  g.J[0][0] = v[2] - v[0];
  g.J[1][0] = v[3] - v[1];
  g.J[0][1] = v[4] - v[0];
  g.J[1][1] = v[5] - v[1];
  for (int k = 0; k < 3; ++k) {  // mesh.py:55-62: outward unit normal of edge k
    const int a = ev[k][0], b = ev[k][1];
    const double tx = v[2 * b] - v[2 * a], ty = v[2 * b + 1] - v[2 * a + 1];
    double nx = ty, ny = -tx;
    if (nx * (v[2 * k] - v[2 * a]) + ny * (v[2 * k + 1] - v[2 * a + 1]) > 0) {
      nx = -nx;
      ny = -ny;
    }
    const double l = sqrt(nx * nx + ny * ny);
    g.nrm[k][0] = nx / l;
    g.nrm[k][1] = ny / l;
    g.len[k] = sqrt(tx * tx + ty * ty);
  }
  // MacroElement.diameter (mesh.py:106-110)
  const double d01 = sqrt((v[0] - v[2]) * (v[0] - v[2]) + (v[1] - v[3]) * (v[1] - v[3]));
  const double d12 = sqrt((v[2] - v[4]) * (v[2] - v[4]) + (v[3] - v[5]) * (v[3] - v[5]));
  const double d20 = sqrt((v[4] - v[0]) * (v[4] - v[0]) + (v[5] - v[1]) * (v[5] - v[1]));
  g.diam = fmax(d01, fmax(d12, d20));
}

__device__ double supg_param(double h, double ax, double ay, double kappa, int plus) {
  const double an = sqrt(ax * ax + ay * ay);  // assembly.py:94-111
  if (an == 0.0) return 0.0;
  const double pe = an * h / (2.0 * kappa);
  const double sign = plus ? 1.0 : -1.0;
  double g;
  if (pe > 30.0) g = 1.0 + sign / pe;
  else if (pe < 1e-4) {
    g = pe / 3.0 - pe * pe * pe / 45.0;
    if (sign > 0) g += 2.0 / pe;
  } else g = 1.0 / tanh(pe) + sign / pe;
  return h / (2.0 * an) * g;
}

// one macro per CTA
__global__ void __launch_bounds__(kAsmThreads) assemble_macro_kernel(AsmDev a) {
  const mh_hdg2d_tables& T = a.T;
  const int nb = T.nb, nq = T.nq, Q = T.Q, t = T.t, nloc = 3 * Q, nc = a.S * t, nb2 = nb * nb;
  extern __shared__ double sm[];
  double* tabs = sm;                       // [2 kinds][4: M, Kx, Ky, S][nb*nb]
  double* gph = tabs + 8 * nb2;            // nq x nb x 2
  double* advg = gph + 2 * nq * nb;        // nq x nb
  double* lap = advg + nq * nb;            // nq x nb
  double* wd = lap + nq * nb;              // [2 kinds][nq]
  double* W = wd + 2 * nq;                 // t x t
  double* Me = W + t * t;                  // t x t
  __shared__ Geo g;
  __shared__ double ts_k[2], Jinv_k[2][2][2];
  const double ax = T.ax, ay = T.ay, kappa = T.kappa;

  for (int64_t e = blockIdx.x; e < a.N; e += gridDim.x) {
    if (threadIdx.x == 0) geometry(a.verts + e * 6, g);
    double* Ae = a.A + e * (int64_t)nloc * nloc;
    double* Be = a.B + e * (int64_t)nloc * nc;
    double* Ce = a.C + e * (int64_t)nc * nloc;
    double* Re = a.Ru + e * (int64_t)nloc;
    for (int64_t i = threadIdx.x; i < (int64_t)nloc * nloc; i += blockDim.x) Ae[i] = 0.0;
    for (int i = threadIdx.x; i < nloc * nc; i += blockDim.x) {
      Be[i] = 0.0;
      Ce[i] = 0.0;
    }
    for (int i = threadIdx.x; i < nloc; i += blockDim.x) Re[i] = 0.0;
    __syncthreads();
    // ---- the two congruence classes of sub-cells (assembly.py:198-218)
    for (int kind = 0; kind < 2; ++kind) {
      if (threadIdx.x == 0) {
        const double m = (double)T.m;
        const double js[2][2] = {{kind ? 0.0 : 1.0 / m, kind ? -1.0 / m : 0.0},
                                 {kind ? 1.0 / m : 0.0, 1.0 / m}};
        double Jc[2][2];
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) Jc[i][j] = g.J[i][0] * js[0][j] + g.J[i][1] * js[1][j];
        const double det = Jc[0][0] * Jc[1][1] - Jc[0][1] * Jc[1][0];
        Jinv_k[kind][0][0] = Jc[1][1] / det;
        Jinv_k[kind][0][1] = -Jc[0][1] / det;
        Jinv_k[kind][1][0] = -Jc[1][0] / det;
        Jinv_k[kind][1][1] = Jc[0][0] / det;
        for (int q = 0; q < nq; ++q) wd[kind * nq + q] = T.qw[q] * fabs(det);
        ts_k[kind] = 0.0;
        if (T.supg) {
          const double e0 = sqrt(Jc[0][0] * Jc[0][0] + Jc[1][0] * Jc[1][0]);
          const double e1 = sqrt(Jc[0][1] * Jc[0][1] + Jc[1][1] * Jc[1][1]);
          const double dx = Jc[0][1] - Jc[0][0], dy = Jc[1][1] - Jc[1][0];
          const double h = fmax(e0, fmax(e1, sqrt(dx * dx + dy * dy)));
          ts_k[kind] = supg_param(h, ax, ay, kappa, T.supg_plus);
        }
      }
      __syncthreads();
      const double(*Ji)[2] = Jinv_k[kind];
      for (int i = threadIdx.x; i < nq * nb; i += blockDim.x) {  // gph = gref @ Jinv
        const double g0 = T.gref[2 * i], g1 = T.gref[2 * i + 1];
        const double p0 = g0 * Ji[0][0] + g1 * Ji[1][0];
        const double p1 = g0 * Ji[0][1] + g1 * Ji[1][1];
        gph[2 * i] = p0;
        gph[2 * i + 1] = p1;
        if (T.supg) {
          advg[i] = p0 * ax + p1 * ay;
          const double* hq = T.href + 4 * i;  // einsum("ja,qbjk,ka->qb", Jinv, href, Jinv)
          double s = 0.0;
          for (int aa = 0; aa < 2; ++aa)
            for (int j = 0; j < 2; ++j)
              for (int k = 0; k < 2; ++k) s += Ji[j][aa] * hq[2 * j + k] * Ji[k][aa];
          lap[i] = s;
        }
      }
      __syncthreads();
      const double* wdk = wd + kind * nq;
      double* tk = tabs + kind * 4 * nb2;
      for (int ij = threadIdx.x; ij < nb2; ij += blockDim.x) {
        const int ia = ij / nb, ib = ij - ia * nb;
        double M = 0.0, K0 = 0.0, K1 = 0.0, Sv = 0.0;
        for (int q = 0; q < nq; ++q) {
          const double vb = T.val[q * nb + ib], w = wdk[q];
          M = fma(T.val[q * nb + ia], w * vb, M);
          K0 = fma(gph[2 * (q * nb + ia)] * w, vb, K0);
          K1 = fma(gph[2 * (q * nb + ia) + 1] * w, vb, K1);
          if (T.supg)
            Sv = fma(advg[q * nb + ia] * w, advg[q * nb + ib] - kappa * lap[q * nb + ib], Sv);
        }
        tk[ij] = M;
        tk[nb2 + ij] = K0;
        tk[2 * nb2 + ij] = K1;
        tk[3 * nb2 + ij] = ts_k[kind] * Sv;
      }
      __syncthreads();
    }
    // ---- scatter over the sub-cells (assembly.py:220-235)
    for (int c = 0; c < T.ncell; ++c) {
      const int kind = T.cell_kind[c];
      const int* cm = T.cell_map + c * nb;
      const double* tk = tabs + kind * 4 * nb2;
      for (int ij = threadIdx.x; ij < nb2; ij += blockDim.x) {
        const int ia = ij / nb, ib = ij - ia * nb;
        const int ra = cm[ia], rb = cm[ib];
        const double M = tk[ij], K0 = tk[nb2 + ij], K1 = tk[2 * nb2 + ij];
        Ae[(int64_t)ra * nloc + rb] += M;
        Ae[(int64_t)(Q + ra) * nloc + Q + rb] += M;
        double* uu = Ae + (int64_t)(2 * Q + ra) * nloc + 2 * Q + rb;
        Ae[(int64_t)ra * nloc + 2 * Q + rb] += -K0;
        Ae[(int64_t)(2 * Q + ra) * nloc + rb] += -kappa * K0;
        *uu += -ax * K0;
        Ae[(int64_t)(Q + ra) * nloc + 2 * Q + rb] += -K1;
        Ae[(int64_t)(2 * Q + ra) * nloc + Q + rb] += -kappa * K1;
        *uu += -ay * K1;
        if (T.supg) *uu += tk[3 * nb2 + ij];
      }
      if ((int)threadIdx.x < nb) {  // load vector: val^T (wd f) [+ ts advg^T (wd f)]
        const int ia = threadIdx.x;
        const double* fv = a.fq + (e * T.ncell + c) * nq;
        const double* wdk = wd + kind * nq;
        double r = 0.0;
        for (int q = 0; q < nq; ++q) r = fma(T.val[q * nb + ia], wdk[q] * fv[q], r);
        double* re = Re + 2 * Q + cm[ia];
        *re += r;
        if (T.supg) {
          const double(*Ji)[2] = Jinv_k[kind];
          double s = 0.0;
          for (int q = 0; q < nq; ++q) {
            const double g0 = T.gref[2 * (q * nb + ia)], g1 = T.gref[2 * (q * nb + ia) + 1];
            const double ad = (g0 * Ji[0][0] + g1 * Ji[1][0]) * ax + (g0 * Ji[0][1] + g1 * Ji[1][1]) * ay;
            s = fma(ad, wdk[q] * fv[q], s);
          }
          *re += ts_k[kind] * s;
        }
      }
      __syncthreads();
    }
    // ---- face terms, one slot per face in the macro's face order (assembly.py:252-283)
    for (int k = 0; k < a.S; ++k) {
      const int edge = a.slot_edge[e * a.S + k];
      if (edge < 0) break;  // no more faces on this macro
      const double n0 = g.nrm[edge][0], n1 = g.nrm[edge][1];
      const double an = ax * n0 + ay * n1;
      const double tau = fabs(an) + kappa / g.diam;  // stabilization_tau (assembly.py:85-91)
      const int var = a.slot_var[e * a.S + k];
      const double* TH = T.th + (int64_t)var * T.nfq * t;
      const double* PS = T.ps + (int64_t)var * T.nfq * t;
      const double* FW = T.fw + (int64_t)var * T.nfq;
      const double lenF = a.slot_len[e * a.S + k];
      for (int ij = threadIdx.x; ij < t * t; ij += blockDim.x) {
        const int i = ij / t, j = ij - i * t;
        double w = 0.0, me = 0.0;
        for (int s = 0; s < T.nfq; ++s) {
          const double wl = FW[s] * lenF;
          w = fma(TH[s * t + i], wl * PS[s * t + j], w);
          me = fma(TH[s * t + i], wl * TH[s * t + j], me);
        }
        W[ij] = w;
        Me[ij] = me;
      }
      __syncthreads();
      const int* en = T.edge_nodes + edge * t;
      for (int ij = threadIdx.x; ij < t * t; ij += blockDim.x) {
        const int i = ij / t, j = ij - i * t;
        const int ri = en[i], rj = en[j];
        const double w = W[ij], me = Me[ij];
        for (int c = 0; c < 2; ++c) {
          const double nc_ = c ? n1 : n0;
          Ae[(int64_t)(2 * Q + ri) * nloc + c * Q + rj] += kappa * nc_ * me;
          Be[(int64_t)(c * Q + ri) * nc + k * t + j] += nc_ * w;
          Ce[(int64_t)(k * t + j) * nloc + c * Q + ri] += kappa * nc_ * w;
        }
        Ae[(int64_t)(2 * Q + ri) * nloc + 2 * Q + rj] += tau * me;
        Be[(int64_t)(2 * Q + ri) * nc + k * t + j] += (an - tau) * w;
        Ce[(int64_t)(k * t + j) * nloc + 2 * Q + ri] += tau * w;
      }
      __syncthreads();
    }
    // ---- Dirichlet trace elimination R_u -= B[:, slot] ghat (assembly.py:285-290)
    for (int k = 0; k < a.S; ++k) {
      const int dk = a.slot_dir[e * a.S + k];
      if (dk < 0) continue;
      const double* gh = a.ghat + (int64_t)dk * t;
      for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < t; ++j) s = fma(Be[(int64_t)i * nc + k * t + j], gh[j], s);
        Re[i] -= s;
      }
      __syncthreads();
    }
  }
}

// D = (sum over the face's sides of a.n - tau) * Mface (assembly.py:293-312);
// one warp per unknown face
__global__ void assemble_face_kernel(mh_hdg2d_tables T, int64_t F, const double* verts,
                                     const int32_t* sides, const double* face_len, double* D) {
  const int lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (f >= F) return;
  const int t = T.t;
  double coef = 0.0;
  const double len = face_len[f];
  for (int sd = 0; sd < 2; ++sd) {
    const int e = sides[f * 4 + 2 * sd], k = sides[f * 4 + 2 * sd + 1];
    if (e < 0) continue;
    Geo g;
    geometry(verts + (int64_t)e * 6, g);
    const double an = T.ax * g.nrm[k][0] + T.ay * g.nrm[k][1];
    const double tau = fabs(an) + T.kappa / g.diam;
    coef += an - tau;
  }
  for (int ij = lane; ij < t * t; ij += 32) {
    const int i = ij / t, j = ij - i * t;
    double m = 0.0;
    for (int s = 0; s < T.nffq; ++s) m = fma(T.fps[s * t + i], T.ffw[s] * len * T.fps[s * t + j], m);
    D[f * t * t + ij] = coef * m;
  }
}

}  // namespace
}  // namespace mh

using namespace mh;

extern "C" int mh_assemble_macros_2d(const mh_hdg2d_tables* tab, int64_t N, int nslot,
                                     const double* verts, const int8_t* slot_edge,
                                     const int8_t* slot_var, const int32_t* slot_dirichlet,
                                     const double* slot_len, const double* ghat,
                                     const double* fq, double* A, double* B, double* C,
                                     double* Ru, void* stream) {
  if (!tab || N < 0 || tab->nb < 1 || tab->nq < 1 || tab->t < 1 || tab->Q < 1 || nslot < 1 ||
      nslot > kMaxSlots) {
    set_error("mh_assemble_macros_2d: bad arguments");
    return MH_E_ARG;
  }
  if (N == 0) return MH_OK;
  if (!verts || !slot_edge || !slot_var || !slot_dirichlet || !slot_len || !fq || !A || !B ||
      !C || !Ru) {
    set_error("mh_assemble_macros_2d: null pointer");
    return MH_E_ARG;
  }
  AsmDev a;
  a.T = *tab;
  a.N = N;
  a.verts = verts;
  a.S = nslot;
  a.slot_edge = slot_edge;
  a.slot_var = slot_var;
  a.slot_dir = slot_dirichlet;
  a.slot_len = slot_len;
  a.ghat = ghat;
  a.fq = fq;
  a.A = A;
  a.B = B;
  a.C = C;
  a.Ru = Ru;
  const int nb = tab->nb, nq = tab->nq, t = tab->t;
  const size_t smem = sizeof(double) * (8 * nb * nb + 4 * nq * nb + 2 * nq + 2 * t * t);
  MH_CHECK_CUDA(cudaFuncSetAttribute(assemble_macro_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 0;
  MH_CHECK_CUDA(cudaGetDevice(&dev));
  MH_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t grid = std::min<int64_t>(N, (int64_t)sms * 16);
  assemble_macro_kernel<<<(unsigned)grid, kAsmThreads, smem, (cudaStream_t)stream>>>(a);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

extern "C" int mh_assemble_faces_2d(const mh_hdg2d_tables* tab, int64_t F, const double* verts,
                                    const int32_t* face_sides, const double* face_len, double* D,
                                    void* stream) {
  if (!tab || F < 0 || tab->t < 1) {
    set_error("mh_assemble_faces_2d: bad arguments");
    return MH_E_ARG;
  }
  if (F == 0) return MH_OK;
  if (!verts || !face_sides || !face_len || !D) {
    set_error("mh_assemble_faces_2d: null pointer");
    return MH_E_ARG;
  }
  const int wpb = 8;
  assemble_face_kernel<<<(unsigned)((F + wpb - 1) / wpb), wpb * 32, 0, (cudaStream_t)stream>>>(
      *tab, F, verts, face_sides, face_len, D);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}
