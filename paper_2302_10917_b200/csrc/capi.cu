// The C-ABI of libmehdg_b200.so: system lifecycle, uploads, factorisation
// and the operator entry points.  See include/mehdg_b200.h for the mapping
// to the reference functions (schur_solver.py).

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <thread>
#include <vector>

#include "mh_internal.h"

namespace mh {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace mh

using namespace mh;

extern "C" const char* mh_last_error(void) { return g_err.c_str(); }
extern "C" int mh_version(void) { return 1; }

extern "C" int mh_device_count(int* count) {
  if (!count) return MH_E_ARG;
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return MH_OK;
}

namespace mh {
static cudaEvent_t take_event(mh_system* s) {
  if (!s->ev_pool.empty()) {
    cudaEvent_t e = s->ev_pool.back();
    s->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
int prof_begin(mh_system* s, cudaEvent_t* ev) {
  *ev = nullptr;
  if (!s->profiling) return MH_OK;
  *ev = take_event(s);
  MH_CHECK_CUDA(cudaEventRecord(*ev, s->stream));
  return MH_OK;
}
int prof_end(mh_system* s, cudaEvent_t ev0, int kind) {
  if (!s->profiling || !ev0) return MH_OK;
  cudaEvent_t ev1 = take_event(s);
  MH_CHECK_CUDA(cudaEventRecord(ev1, s->stream));
  (kind == 0 ? s->ev_elem : s->ev_face).emplace_back(ev0, ev1);
  return MH_OK;
}
}  // namespace mh

extern "C" int mh_profile(mh_system* s, int enable) {
  if (!s) return MH_E_ARG;
  s->profiling = enable != 0;
  return MH_OK;
}

extern "C" int mh_profile_read(mh_system* s, double* elem_ms, int64_t* elem_n, double* face_ms,
                               int64_t* face_n) {
  if (!s) return MH_E_ARG;
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  double sums[2] = {0.0, 0.0};
  int64_t counts[2] = {0, 0};
  for (int k = 0; k < 2; ++k) {
    auto& v = k == 0 ? s->ev_elem : s->ev_face;
    for (auto& pr : v) {
      float ms = 0.f;
      MH_CHECK_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      sums[k] += ms;
      counts[k] += 1;
      s->ev_pool.push_back(pr.first);
      s->ev_pool.push_back(pr.second);
    }
    v.clear();
  }
  if (elem_ms) *elem_ms = sums[0];
  if (elem_n) *elem_n = counts[0];
  if (face_ms) *face_ms = sums[1];
  if (face_n) *face_n = counts[1];
  return MH_OK;
}

static int need(mh_system* s, bool cond, const char* msg) {
  if (!s) {
    set_error("null system");
    return MH_E_ARG;
  }
  if (!cond) {
    set_error(msg);
    return MH_E_STATE;
  }
  return MH_OK;
}

namespace mh {
int launch_occupancy(int device, const void* kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> attr;           // smem attribute set
  static std::map<std::tuple<int, const void*, int, size_t>, int> occ;  // resident CTAs / SM
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(device, kern, threads, smem);
  auto it = occ.find(key);
  if (it != occ.end()) return it->second;
  size_t& cur = attr[{device, kern}];
  if (smem > cur) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      return -1;
    }
    cur = smem;
  }
  int per_sm = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (e != cudaSuccess) {
    set_error(std::string("cudaOccupancyMaxActiveBlocksPerMultiprocessor: ") + cudaGetErrorString(e));
    return -1;
  }
  occ[key] = per_sm;
  return per_sm;
}

void Knobs::read() {
  auto env = [](const char* k) { return getenv(k); };
  if (const char* v = env("MEHDG_LU")) lu = !strcmp(v, "tile") ? 1 : (!strcmp(v, "cta") ? 2 : (!strcmp(v, "pipe") ? 3 : 0));
  if (const char* v = env("MEHDG_LU_PIPE_W")) lu_pipe_w = atoi(v);
  if (const char* v = env("MEHDG_LU_PIPE_CTAS")) lu_pipe_ctas = atoi(v);
  if (const char* v = env("MEHDG_LU_CTAS")) lu_ctas = std::max(1, atoi(v));
  if (const char* v = env("MEHDG_LU_SCR")) lu_scr_pol = atoi(v);
  if (const char* v = env("MEHDG_LU_APOL")) lu_a_pol = atoi(v);
  if (const char* v = env("MEHDG_ELEM_CTAS")) elem_ctas = std::max(0, atoi(v));
  if (const char* v = env("MEHDG_ELEM_CH")) elem_ch = atoi(v);
  if (const char* v = env("MEHDG_ELEM_BPOL")) elem_bpol = atoi(v);
  if (const char* v = env("MEHDG_ELEM_LPOL")) elem_lpol = atoi(v);
  if (const char* v = env("MEHDG_MB_STREAM")) mb_stream = atoi(v);
  if (const char* v = env("MEHDG_ELEM_SPLIT")) elem_split = atoi(v);
  if (const char* v = env("MEHDG_ELEM_SPLIT_CTAS")) elem_split_ctas = atoi(v);
  if (const char* v = env("MEHDG_MGS_SMALL")) mgs_small = atoi(v);
  if (const char* v = env("MEHDG_MGS_CTAS")) mgs_ctas = std::max(1, atoi(v));
  if (const char* v = env("MEHDG_MGS_REG")) mgs_reg = atoi(v);
  if (const char* v = env("MEHDG_FACE_BULK")) face_bulk = atoi(v);
  if (const char* v = env("MEHDG_GMRES_GRAPHS")) gmres_graphs = atoi(v);
  if (const char* v = env("MEHDG_SPLIT_AT")) split_at = atoll(v);
}
}  // namespace mh

extern "C" int mh_create(int device, int nfe, int64_t n_elem, int q, int t, int64_t n_face,
                         mh_system** out) {
  if (!out || nfe < 1 || nfe > kMaxSlots || n_elem < 0 || q < 1 || t < 1 || n_face < 0) {
    set_error("mh_create: bad sizes");
    return MH_E_ARG;
  }
  if (q > 256 || t > 128) {
    set_error("mh_create: Q <= 256 and t <= 128 are supported");
    return MH_E_UNSUPPORTED;
  }
  *out = nullptr;
  MH_CHECK_CUDA(cudaSetDevice(device));
  mh_system* s = new mh_system();
  s->knobs.read();
  s->device = device;
  s->nfe = nfe;
  s->N = n_elem;
  s->Q = q;
  s->t = t;
  s->nc = nfe * t;
  s->F = n_face;
  cudaDeviceGetAttribute(&s->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete s;
    set_error(std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    return MH_E_CUDA;
  }
  s->own_stream = true;
  *out = s;
  return MH_OK;
}

extern "C" int mh_destroy(mh_system* s) {
  if (!s) return MH_OK;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  s->elem_ufac.release(); s->face_vslot.release();
  s->A.release(); s->lu_scr.release(); s->lu_fb.release(); s->Lp.release(); s->Up.release(); s->udiag.release();
  s->dinv.release(); s->piv.release(); s->perm.release();
  s->lstat.release(); s->Bt.release(); s->Cm.release(); s->Ru.release(); s->D.release();
  s->Draw.release(); s->Rhat.release(); s->Dinv.release(); s->Fkind.release(); s->V.release();
  s->tmp.release(); s->S.release(); s->halo_u.release(); s->hin.release(); s->hout.release();
  if (s->kry) free_krylov(s->kry);
  free_comm(s);
  for (auto& pr : s->ev_elem) { s->ev_pool.push_back(pr.first); s->ev_pool.push_back(pr.second); }
  for (auto& pr : s->ev_face) { s->ev_pool.push_back(pr.first); s->ev_pool.push_back(pr.second); }
  for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
  if (s->cin) {
    cudaStreamDestroy(s->cin);
    cudaStreamDestroy(s->cout);
    for (cudaEvent_t e : s->evp) cudaEventDestroy(e);
  }
  if (s->kstream) {
    cudaStreamDestroy(s->kstream);
    cudaEventDestroy(s->ev_u);
    cudaEventDestroy(s->ev_int);
  }
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return MH_OK;
}

extern "C" int mh_set_stream(mh_system* s, void* stream) {
  if (!s) return MH_E_ARG;
  if (s->own_stream && s->stream) {
    cudaStreamSynchronize(s->stream);
    cudaStreamDestroy(s->stream);
  }
  s->stream = (cudaStream_t)stream;
  s->own_stream = false;
  return MH_OK;
}

extern "C" int mh_upload_connectivity(mh_system* s, const int32_t* elem_ufac,
                                      const int32_t* face_elem, const int32_t* face_slot) {
  if (!s || (s->N > 0 && !elem_ufac) || (s->F > 0 && (!face_elem || !face_slot))) {
    set_error("mh_upload_connectivity: null argument");
    return MH_E_ARG;
  }
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  const int64_t ntrace = s->F + s->F_halo;
  s->e_split = 0;  // one past the last macro that reads a received halo trace
  for (int64_t i = 0; i < s->N * s->nfe; ++i) {
    if (elem_ufac[i] < -1 || elem_ufac[i] >= ntrace) {
      set_error("elem_ufac entry out of range");
      return MH_E_ARG;
    }
    if (elem_ufac[i] >= s->F) s->e_split = i / s->nfe + 1;
  }
  std::vector<int32_t> vslot((size_t)(2 * s->F));
  for (int64_t f = 0; f < s->F; ++f)
    for (int c = 0; c < 2; ++c) {
      const int32_t e = face_elem[2 * f + c], k = face_slot[2 * f + c];
      if (e < 0) {
        vslot[2 * f + c] = -1;
        continue;
      }
      if (e >= s->N + s->n_vslot_extra || k < 0 || k >= s->nfe) {
        set_error("face table entry out of range");
        return MH_E_ARG;
      }
      // e >= N addresses a received v-slot segment (multi-GPU halo)
      vslot[2 * f + c] = e < s->N ? (int32_t)(e * s->nfe + k)
                                  : (int32_t)(s->N * s->nfe + (e - s->N));
    }
  s->h_face_elem.assign(face_elem, face_elem + 2 * s->F);
  s->h_face_slot.assign(face_slot, face_slot + 2 * s->F);
  MH_CHECK(s->elem_ufac.alloc((size_t)(s->N * s->nfe)));
  MH_CHECK(s->face_vslot.alloc((size_t)(2 * s->F)));
  if (s->N)
    MH_CHECK_CUDA(cudaMemcpyAsync(s->elem_ufac.p, elem_ufac, sizeof(int32_t) * s->N * s->nfe,
                                  cudaMemcpyHostToDevice, s->stream));
  if (s->F)
    MH_CHECK_CUDA(cudaMemcpyAsync(s->face_vslot.p, vslot.data(), sizeof(int32_t) * 2 * s->F,
                                  cudaMemcpyHostToDevice, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  s->have_conn = true;
  return MH_OK;
}

static int alloc_blocks(mh_system* s) {
  const size_t N = (size_t)s->N, Q = s->Q, nc = s->nc, F = (size_t)s->F, t = s->t;
  const int64_t ch = kStreamChunk;
  s->ldB = ((int64_t)nc * Q + ch - 1) / ch * ch;
  s->ldL = ((int64_t)Q * (Q - 1) / 2 + ch - 1) / ch * ch;
  if (s->ldL < ch) s->ldL = ch;
  MH_CHECK(s->A.alloc(N * Q * Q));
  MH_CHECK(s->Lp.alloc(N * (size_t)s->ldL));
  MH_CHECK(s->Up.alloc(N * (size_t)s->ldL));
  MH_CHECK(s->udiag.alloc(N * Q));
  MH_CHECK(s->dinv.alloc(N * Q));
  MH_CHECK(s->piv.alloc(N * Q));
  MH_CHECK(s->perm.alloc(N * Q));
  MH_CHECK(s->lstat.alloc(N));
  MH_CHECK(s->Bt.alloc(N * (size_t)s->ldB));
  MH_CHECK(s->Ru.alloc(N * Q));
  s->ldF = ((int64_t)t * t + 1) & ~int64_t(1);
  MH_CHECK(s->D.alloc(F * s->ldF));
  MH_CHECK(s->Draw.alloc(F * t * t));
  MH_CHECK(s->Rhat.alloc(F * t));
  MH_CHECK(s->Dinv.alloc(F * s->ldF));
  MH_CHECK(s->Fkind.alloc(F));
  MH_CHECK(s->V.alloc((N * s->nfe + (size_t)s->n_vslot_extra) * t));
  MH_CHECK(s->tmp.alloc((F + (size_t)s->F_halo) * t + 1));
  return MH_OK;
}

// ---- host -> device uploads of the (GB-sized) blocks -------------------------
// A pageable cudaMemcpy runs at host-memcpy speed through the driver's single
// staging thread.  Large uploads instead go through pinned staging buffers:
// T host threads each copy their contiguous slice chunk by chunk into two pinned
// buffers of their own and issue the H2D copies on their own stream, so the
// CPU copies of chunk i+1 overlap the PCIe transfer of chunk i.  The pinned
// buffers, streams and events are created once per device and kept.
namespace {
constexpr size_t kStageChunk = (size_t)4 << 20;
constexpr size_t kStageMin = (size_t)32 << 20;  // below this: plain cudaMemcpyAsync
struct HostStage {
  std::mutex mu;
  int nthr = 0;
  std::vector<void*> buf;        // 2 per thread
  std::vector<cudaStream_t> st;  // 1 per thread
  std::vector<cudaEvent_t> ev;   // 2 per thread
};
HostStage g_stage[16];

int stage_init(HostStage& hs, int device) {
  if (hs.nthr) return MH_OK;
  const unsigned hc = std::thread::hardware_concurrency();
  int n = (int)std::max(1u, std::min(16u, hc ? hc : 1u));
  if (const char* v = getenv("MEHDG_UPLOAD_THREADS")) n = std::max(1, std::min(32, atoi(v)));
  MH_CHECK_CUDA(cudaSetDevice(device));
  hs.st.assign(n, nullptr);
  hs.buf.assign(2 * n, nullptr);
  hs.ev.assign(2 * n, nullptr);
  // page-locking is the slow part of the first upload: the threads do it in parallel
  std::vector<cudaError_t> res(n, cudaSuccess);
  auto mk = [&](int i) {
    cudaError_t ce = cudaSetDevice(device);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&hs.st[i], cudaStreamNonBlocking);
    for (int b = 0; b < 2 && ce == cudaSuccess; ++b) {
      ce = cudaHostAlloc(&hs.buf[2 * i + b], kStageChunk, cudaHostAllocDefault);
      if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&hs.ev[2 * i + b], cudaEventDisableTiming);
    }
    res[i] = ce;
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n; ++i) th.emplace_back(mk, i);
  mk(0);
  for (auto& x : th) x.join();
  for (int i = 0; i < n; ++i) MH_CHECK_CUDA(res[i]);
  hs.nthr = n;
  return MH_OK;
}
}  // namespace

// bytes from host memory `src` to device memory `dst`; returns after the copy
// has completed (earlier work on the system stream is drained first)
static int h2d(mh_system* s, void* dst, const void* src, size_t bytes) {
  if (!bytes) return MH_OK;
  static const bool staged = !(getenv("MEHDG_UPLOAD_STAGE") && atoi(getenv("MEHDG_UPLOAD_STAGE")) == 0);
  if (!staged || bytes < kStageMin || s->device < 0 || s->device >= 16) {
    MH_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s->stream));
    MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
    return MH_OK;
  }
  HostStage& hs = g_stage[s->device];
  std::lock_guard<std::mutex> lk(hs.mu);
  MH_CHECK(stage_init(hs, s->device));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  const int n = hs.nthr;
  const size_t per = ((bytes + n - 1) / n + 4095) & ~(size_t)4095;
  std::vector<int> status((size_t)n, MH_OK);
  std::vector<std::string> err((size_t)n);
  auto work = [&](int i) {
    cudaSetDevice(s->device);
    const size_t b0 = std::min(bytes, (size_t)i * per), b1 = std::min(bytes, b0 + per);
    int k = 0;
    for (size_t off = b0; off < b1; off += kStageChunk, ++k) {
      const size_t len = std::min(kStageChunk, b1 - off);
      const int b = k & 1;
      cudaError_t ce = cudaSuccess;
      if (k >= 2) ce = cudaEventSynchronize(hs.ev[2 * i + b]);
      if (ce == cudaSuccess) {
        std::memcpy(hs.buf[2 * i + b], static_cast<const char*>(src) + off, len);
        ce = cudaMemcpyAsync(static_cast<char*>(dst) + off, hs.buf[2 * i + b], len,
                             cudaMemcpyHostToDevice, hs.st[i]);
      }
      if (ce == cudaSuccess) ce = cudaEventRecord(hs.ev[2 * i + b], hs.st[i]);
      if (ce != cudaSuccess) {
        status[i] = MH_E_CUDA;
        err[i] = cudaGetErrorString(ce);
        return;
      }
    }
    const cudaError_t ce = cudaStreamSynchronize(hs.st[i]);
    if (ce != cudaSuccess) {
      status[i] = MH_E_CUDA;
      err[i] = cudaGetErrorString(ce);
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n; ++i) th.emplace_back(work, i);
  work(0);
  for (auto& x : th) x.join();
  for (int i = 0; i < n; ++i)
    if (status[i] != MH_OK) {
      set_error("staged upload: " + err[i]);
      return status[i];
    }
  return MH_OK;
}

static int upload_impl(mh_system* s, const double* A, const double* B, const double* C,
                       const double* Ru, const double* D, const double* Rhat,
                       cudaMemcpyKind kind) {
  if (!s || (s->N > 0 && !A) || (s->N > 0 && !B && !C) || (s->F > 0 && !D)) {
    set_error("mh_upload_blocks: null argument");
    return MH_E_ARG;
  }
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  MH_CHECK(alloc_blocks(s));
  const size_t N = (size_t)s->N, Q = s->Q, nc = s->nc, F = (size_t)s->F, t = s->t;
  cudaStream_t st = s->stream;
  const bool host = kind == cudaMemcpyHostToDevice;
  // contiguous copies: staged through pinned buffers from host memory
  auto copy = [&](void* dst, const void* src, size_t bytes) -> int {
    if (host) return h2d(s, dst, src, bytes);
    if (bytes) MH_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, st));
    return MH_OK;
  };
  if (N) MH_CHECK(copy(s->A.p, A, sizeof(double) * N * Q * Q));
  s->c_is_bt = (B == nullptr) || (C == nullptr);
  if (!s->c_is_bt) MH_CHECK(s->Cm.alloc(N * (size_t)s->ldB));
  else s->Cm.release();
  const size_t row = sizeof(double) * nc * Q, pitch = sizeof(double) * (size_t)s->ldB;
  if (N && (size_t)s->ldB != nc * Q)  // zero the per-macro pad (streamed, never used)
    MH_CHECK_CUDA(cudaMemsetAsync(s->Bt.p, 0, pitch * N, st));
  // a (N x rows) block with host row length `row` into device pitch `pitch`:
  // contiguous upload to the staging buffer, then a device-side pitched copy
  auto copy_pitched = [&](double* dst, const double* src) -> int {
    if (!host) {
      MH_CHECK_CUDA(cudaMemcpy2DAsync(dst, pitch, src, row, row, N, kind, st));
      return MH_OK;
    }
    MH_CHECK(s->S.alloc(N * nc * Q));
    MH_CHECK(h2d(s, s->S.p, src, row * N));
    MH_CHECK_CUDA(cudaMemcpy2DAsync(dst, pitch, s->S.p, row, row, N, cudaMemcpyDeviceToDevice, st));
    MH_CHECK_CUDA(cudaStreamSynchronize(st));
    s->S.release();
    return MH_OK;
  };
  if (B == nullptr) {
    if (N) MH_CHECK(copy_pitched(s->Bt.p, C));
  } else {
    // op.B (N x Q x nc) -> Bt (N x nc x Q, stride ldB) through a staging buffer
    if (N) {
      MH_CHECK(s->S.alloc(N * nc * Q));
      MH_CHECK(copy(s->S.p, B, row * N));
      MH_CHECK(launch_transpose_batched(st, s->S.p, s->Bt.p, (int64_t)N, (int)Q, (int)nc,
                                        s->ldB));
      MH_CHECK_CUDA(cudaStreamSynchronize(st));
      s->S.release();
    }
    if (C && N) {
      MH_CHECK_CUDA(cudaMemsetAsync(s->Cm.p, 0, pitch * N, st));
      MH_CHECK(copy_pitched(s->Cm.p, C));
    }
  }
  if (N) {
    if (Ru) MH_CHECK(copy(s->Ru.p, Ru, sizeof(double) * N * Q));
    else MH_CHECK_CUDA(cudaMemsetAsync(s->Ru.p, 0, sizeof(double) * N * Q, st));
  }
  if (F) {
    MH_CHECK(copy(s->Draw.p, D, sizeof(double) * F * t * t));
    if (Rhat) MH_CHECK(copy(s->Rhat.p, Rhat, sizeof(double) * F * t));
    else MH_CHECK_CUDA(cudaMemsetAsync(s->Rhat.p, 0, sizeof(double) * F * t, st));
  }
  MH_CHECK_CUDA(cudaMemsetAsync(s->V.p, 0, sizeof(double) * s->V.n, st));
  MH_CHECK_CUDA(cudaStreamSynchronize(st));
  s->have_blocks = true;
  s->factored = false;
  s->have_mb = false;
  return MH_OK;
}

extern "C" int mh_upload_blocks(mh_system* s, const double* A, const double* B, const double* C,
                                const double* Ru, const double* D, const double* Rhat) {
  return upload_impl(s, A, B, C, Ru, D, Rhat, cudaMemcpyHostToDevice);
}

extern "C" int mh_upload_blocks_device(mh_system* s, const double* A, const double* B,
                                       const double* C, const double* Ru, const double* D,
                                       const double* Rhat) {
  return upload_impl(s, A, B, C, Ru, D, Rhat, cudaMemcpyDeviceToDevice);
}

extern "C" int mh_factorize(mh_system* s, int32_t* fail_macro, int32_t* fail_face,
                            int8_t* face_kinds, float* lu_ms) {
  MH_CHECK(need(s, s && s->have_blocks, "mh_factorize before mh_upload_blocks"));
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  if (fail_macro) *fail_macro = -1;
  if (fail_face) *fail_face = -1;
  MH_CHECK(launch_lu(s, lu_ms));
  MH_CHECK(launch_face_factor(s, s->Draw.p));
  std::vector<int32_t> st((size_t)s->N);
  std::vector<int8_t> kinds((size_t)s->F);
  if (s->N)
    MH_CHECK_CUDA(cudaMemcpyAsync(st.data(), s->lstat.p, sizeof(int32_t) * s->N,
                                  cudaMemcpyDeviceToHost, s->stream));
  if (s->F)
    MH_CHECK_CUDA(cudaMemcpyAsync(kinds.data(), s->Fkind.p, s->F, cudaMemcpyDeviceToHost,
                                  s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  if (face_kinds && s->F) std::memcpy(face_kinds, kinds.data(), s->F);
  // the reference factorises all macros before any face (schur_solver.py:195-196)
  for (int64_t e = 0; e < s->N; ++e)
    if (st[e]) {
      if (fail_macro) *fail_macro = (int32_t)e;
      set_error("singular local block");
      return MH_E_SINGULAR_LOCAL;
    }
  for (int64_t f = 0; f < s->F; ++f)
    if (kinds[f] == MH_FACE_SINGULAR) {
      if (fail_face) *fail_face = (int32_t)f;
      set_error("singular face block");
      return MH_E_SINGULAR_FACE;
    }
  s->factored = true;
  return MH_OK;
}

extern "C" int mh_refactorize_local(mh_system* s, float* lu_ms) {
  MH_CHECK(need(s, s && s->have_blocks, "mh_refactorize_local before upload"));
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  return launch_lu(s, lu_ms);
}

// The explicit face inverses the preconditioner applies (sign folded in):
// n faces (unknown-face indices idx[]), t x t row-major on the host.  The
// device keeps them column-major (face.cu).
static int face_inverse_io(mh_system* s, int64_t n, const int32_t* idx, double* host, bool set) {
  MH_CHECK(need(s, s && s->factored, "face inverses before mh_factorize"));
  if (n < 0 || (n && (!idx || !host))) {
    set_error("mh_{get,set}_face_inverse: bad arguments");
    return MH_E_ARG;
  }
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  const int t = s->t;
  const size_t TT = (size_t)t * t;
  std::vector<double> cm(TT);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t f = idx[k];
    if (f < 0 || f >= s->F) {
      set_error("mh_{get,set}_face_inverse: face index out of range");
      return MH_E_ARG;
    }
    double* hb = host + k * TT;
    if (set) {
      for (int i = 0; i < t; ++i)
        for (int j = 0; j < t; ++j) cm[(size_t)j * t + i] = hb[(size_t)i * t + j];
      MH_CHECK_CUDA(cudaMemcpyAsync(s->Dinv.p + f * s->ldF, cm.data(), sizeof(double) * TT,
                                    cudaMemcpyHostToDevice, s->stream));
      MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
    } else {
      MH_CHECK_CUDA(cudaMemcpyAsync(cm.data(), s->Dinv.p + f * s->ldF, sizeof(double) * TT,
                                    cudaMemcpyDeviceToHost, s->stream));
      MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
      for (int i = 0; i < t; ++i)
        for (int j = 0; j < t; ++j) hb[(size_t)i * t + j] = cm[(size_t)j * t + i];
    }
  }
  return MH_OK;
}

extern "C" int mh_get_face_inverse(mh_system* s, int64_t n, const int32_t* idx, double* inv_host) {
  return face_inverse_io(s, n, idx, inv_host, false);
}

extern "C" int mh_set_face_inverse(mh_system* s, int64_t n, const int32_t* idx,
                                   const double* inv_host) {
  return face_inverse_io(s, n, idx, const_cast<double*>(inv_host), true);
}

extern "C" int mh_get_local_factors(mh_system* s, int64_t first, int64_t count, double* lu_host,
                                    int32_t* piv_host) {
  MH_CHECK(need(s, s && s->factored, "factors requested before mh_factorize"));
  if (first < 0 || count < 0 || first + count > s->N) {
    set_error("macro range out of bounds");
    return MH_E_ARG;
  }
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  const size_t QQ = (size_t)s->Q * s->Q;
  if (lu_host && count) {
    DBuf<double> tmp;
    MH_CHECK(tmp.alloc(QQ * count));
    // packed device factors -> row-major host (scipy's lu[i, j])
    MH_CHECK(launch_unpack_lu(s, first, count, tmp.p));
    MH_CHECK_CUDA(cudaMemcpyAsync(lu_host, tmp.p, sizeof(double) * QQ * count,
                                  cudaMemcpyDeviceToHost, s->stream));
    MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
    tmp.release();
  }
  if (piv_host && count)
    MH_CHECK_CUDA(cudaMemcpyAsync(piv_host, s->piv.p + first * s->Q,
                                  sizeof(int32_t) * s->Q * count, cudaMemcpyDeviceToHost,
                                  s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  return MH_OK;
}

// ---- operator ---------------------------------------------------------------

static int ready(mh_system* s) {
  MH_CHECK(need(s, s && s->have_conn, "connectivity not uploaded"));
  MH_CHECK(need(s, s->factored, "system not factorised (mh_factorize)"));
  return MH_OK;
}

extern "C" int mh_rhs(mh_system* s, double* f) {
  MH_CHECK(ready(s));
  MH_CHECK(halo_rhs_begin(s));
  MH_CHECK(launch_element(s, kRhs, nullptr, s->V.p));
  MH_CHECK(halo_v_exchange(s));
  return launch_face_reduce(s, nullptr, f, 1, 0);
}

// Element phase of an apply: the uhat halo exchange, then the element kernel.
// On a multi-rank system the macros that read no received trace, [e_split, N),
// run on a second stream while the halo exchange is in flight on the system
// stream; the macros [0, e_split) follow the exchange (overlap the
// interior-macro work with the halo).  Each macro's arithmetic is unchanged, so
// the result is bitwise the same.  MEHDG_SPLIT_AT=k moves the split to k (tests),
// clamped to [e_split, N]: a smaller split would let halo-reading macros run
// before the exchange.
static int apply_elements(mh_system* s, const double* u) {
  int64_t split = s->e_split;
  if (s->knobs.split_at >= 0) split = std::min<int64_t>(s->N, std::max<int64_t>(s->e_split, s->knobs.split_at));
  if (!multi_rank(s) || split >= s->N) {
    MH_CHECK(halo_u_exchange(s, u, nullptr));
    return launch_element(s, kApply, u, s->V.p);
  }
  if (!s->kstream) {
    MH_CHECK_CUDA(cudaStreamCreateWithFlags(&s->kstream, cudaStreamNonBlocking));
    MH_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_u, cudaEventDisableTiming));
    MH_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_int, cudaEventDisableTiming));
  }
  // everything earlier on the system stream (u, and the previous apply's use of
  // V) precedes the interior macros; the exchange is enqueued first so that its
  // NCCL kernel is resident before the persistent element grid fills the SMs
  MH_CHECK_CUDA(cudaEventRecord(s->ev_u, s->stream));
  MH_CHECK(halo_u_exchange(s, u, nullptr));
  MH_CHECK_CUDA(cudaStreamWaitEvent(s->kstream, s->ev_u, 0));
  MH_CHECK(launch_element_range(s, kApply, u, s->V.p, s->kstream, split, s->N));
  MH_CHECK_CUDA(cudaEventRecord(s->ev_int, s->kstream));
  MH_CHECK(launch_element_range(s, kApply, u, s->V.p, s->stream, 0, split));
  MH_CHECK_CUDA(cudaStreamWaitEvent(s->stream, s->ev_int, 0));
  return MH_OK;
}

extern "C" int mh_apply(mh_system* s, const double* u, double* w) {
  MH_CHECK(ready(s));
  cudaEvent_t ev;
  MH_CHECK(prof_begin(s, &ev));
  MH_CHECK(apply_elements(s, u));
  MH_CHECK(prof_end(s, ev, 0));
  MH_CHECK(halo_v_exchange(s));
  MH_CHECK(prof_begin(s, &ev));
  MH_CHECK(launch_face_reduce(s, u, w, 0, 0));
  return prof_end(s, ev, 1);
}

extern "C" int mh_apply_precond(mh_system* s, const double* u, double* z) {
  MH_CHECK(ready(s));
  cudaEvent_t ev;
  MH_CHECK(prof_begin(s, &ev));
  MH_CHECK(apply_elements(s, u));
  MH_CHECK(prof_end(s, ev, 0));
  MH_CHECK(halo_v_exchange(s));
  MH_CHECK(prof_begin(s, &ev));
  MH_CHECK(launch_face_reduce(s, u, z, 0, 1));
  return prof_end(s, ev, 1);
}

extern "C" int mh_precond(mh_system* s, const double* w, double* z) {
  MH_CHECK(ready(s));
  return launch_precond(s, w, z);
}

extern "C" int mh_reconstruct(mh_system* s, const double* u, double* U) {
  MH_CHECK(ready(s));
  MH_CHECK(halo_u_exchange(s, u, nullptr));
  return launch_element(s, kRecon, u, U);
}

static int host_io(mh_system* s, size_t nin, size_t nout) {
  MH_CHECK(s->hin.alloc(std::max<size_t>(nin, 1)));
  MH_CHECK(s->hout.alloc(std::max<size_t>(nout, 1)));
  return MH_OK;
}

extern "C" int mh_apply_host(mh_system* s, const double* u, double* w) {
  MH_CHECK(ready(s));
  const size_t n = (size_t)(s->F * s->t);
  MH_CHECK(host_io(s, n, n));
  MH_CHECK_CUDA(cudaMemcpyAsync(s->hin.p, u, n * 8, cudaMemcpyHostToDevice, s->stream));
  MH_CHECK(mh_apply(s, s->hin.p, s->hout.p));
  MH_CHECK_CUDA(cudaMemcpyAsync(w, s->hout.p, n * 8, cudaMemcpyDeviceToHost, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  return MH_OK;
}

// k host vectors through the operator with the transfers overlapped: vector i
// is copied in on one copy stream while vector i-1 is applied on the system
// stream and vector i-2's result is copied out on another (two device buffer
// pairs; the copy engines run concurrently with the kernels).  Strides are in
// doubles; a zero stride reuses one input / overwrites one output.
extern "C" int mh_apply_host_many(mh_system* s, int64_t k, const double* u, int64_t ldu,
                                  double* w, int64_t ldw) {
  MH_CHECK(ready(s));
  const size_t n = (size_t)(s->F * s->t);
  if (k < 0 || ldu < 0 || ldw < 0 || (k > 0 && (!u || !w))) {
    set_error("mh_apply_host_many: bad arguments");
    return MH_E_ARG;
  }
  if (k == 0) return MH_OK;
  MH_CHECK(host_io(s, 2 * n, 2 * n));
  if (!s->cin) {
    MH_CHECK_CUDA(cudaStreamCreateWithFlags(&s->cin, cudaStreamNonBlocking));
    MH_CHECK_CUDA(cudaStreamCreateWithFlags(&s->cout, cudaStreamNonBlocking));
    for (int b = 0; b < 7; ++b) MH_CHECK_CUDA(cudaEventCreateWithFlags(&s->evp[b], cudaEventDisableTiming));
  }
  cudaEvent_t* ev_in = s->evp;       // [2] copy-in done
  cudaEvent_t* ev_comp = s->evp + 2; // [2] apply done
  cudaEvent_t* ev_out = s->evp + 4;  // [2] copy-out done
  // earlier work on the system stream (which may still read hin / hout) first
  MH_CHECK_CUDA(cudaEventRecord(s->evp[6], s->stream));
  MH_CHECK_CUDA(cudaStreamWaitEvent(s->cin, s->evp[6], 0));
  MH_CHECK_CUDA(cudaStreamWaitEvent(s->cout, s->evp[6], 0));
  for (int64_t i = 0; i < k; ++i) {
    const int b = (int)(i & 1);
    double* ud = s->hin.p + b * n;
    double* wd = s->hout.p + b * n;
    if (i >= 2) MH_CHECK_CUDA(cudaStreamWaitEvent(s->cin, ev_comp[b], 0));
    MH_CHECK_CUDA(cudaMemcpyAsync(ud, u + i * ldu, n * 8, cudaMemcpyHostToDevice, s->cin));
    MH_CHECK_CUDA(cudaEventRecord(ev_in[b], s->cin));
    MH_CHECK_CUDA(cudaStreamWaitEvent(s->stream, ev_in[b], 0));
    if (i >= 2) MH_CHECK_CUDA(cudaStreamWaitEvent(s->stream, ev_out[b], 0));
    MH_CHECK(mh_apply(s, ud, wd));
    MH_CHECK_CUDA(cudaEventRecord(ev_comp[b], s->stream));
    MH_CHECK_CUDA(cudaStreamWaitEvent(s->cout, ev_comp[b], 0));
    MH_CHECK_CUDA(cudaMemcpyAsync(w + i * ldw, wd, n * 8, cudaMemcpyDeviceToHost, s->cout));
    MH_CHECK_CUDA(cudaEventRecord(ev_out[b], s->cout));
  }
  MH_CHECK_CUDA(cudaStreamSynchronize(s->cout));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->cin));
  // the system stream's later work sees hin / hout free again
  MH_CHECK_CUDA(cudaStreamWaitEvent(s->stream, ev_out[(k - 1) & 1], 0));
  return MH_OK;
}

extern "C" int mh_precond_host(mh_system* s, const double* w, double* z) {
  MH_CHECK(ready(s));
  const size_t n = (size_t)(s->F * s->t);
  MH_CHECK(host_io(s, n, n));
  MH_CHECK_CUDA(cudaMemcpyAsync(s->hin.p, w, n * 8, cudaMemcpyHostToDevice, s->stream));
  MH_CHECK(mh_precond(s, s->hin.p, s->hout.p));
  MH_CHECK_CUDA(cudaMemcpyAsync(z, s->hout.p, n * 8, cudaMemcpyDeviceToHost, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  return MH_OK;
}

extern "C" int mh_rhs_host(mh_system* s, double* f) {
  MH_CHECK(ready(s));
  const size_t n = (size_t)(s->F * s->t);
  MH_CHECK(host_io(s, 1, n));
  MH_CHECK(mh_rhs(s, s->hout.p));
  MH_CHECK_CUDA(cudaMemcpyAsync(f, s->hout.p, n * 8, cudaMemcpyDeviceToHost, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  return MH_OK;
}

extern "C" int mh_reconstruct_host(mh_system* s, const double* u, double* U) {
  MH_CHECK(ready(s));
  const size_t n = (size_t)(s->F * s->t), nU = (size_t)s->N * s->Q;
  MH_CHECK(host_io(s, n, nU));
  MH_CHECK_CUDA(cudaMemcpyAsync(s->hin.p, u, n * 8, cudaMemcpyHostToDevice, s->stream));
  MH_CHECK(mh_reconstruct(s, s->hin.p, s->hout.p));
  MH_CHECK_CUDA(cudaMemcpyAsync(U, s->hout.p, nU * 8, cudaMemcpyDeviceToHost, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  return MH_OK;
}

// ---- explicit element Schur (mode "mb") --------------------------------------

extern "C" int mh_form_element_schur(mh_system* s) {
  MH_CHECK(ready(s));
  s->ldS = ((int64_t)s->nc * s->nc + kStreamChunk - 1) / kStreamChunk * kStreamChunk;
  MH_CHECK(s->S.alloc((size_t)s->N * (size_t)s->ldS));
  if ((int64_t)s->nc * s->nc != s->ldS)  // the per-macro pad is streamed, never used
    MH_CHECK_CUDA(cudaMemsetAsync(s->S.p, 0, sizeof(double) * (size_t)s->N * (size_t)s->ldS, s->stream));
  MH_CHECK(launch_element_schur(s));
  s->have_mb = true;
  return MH_OK;
}

extern "C" int mh_apply_mb(mh_system* s, const double* u, double* w) {
  MH_CHECK(ready(s));
  MH_CHECK(need(s, s->have_mb, "mh_apply_mb before mh_form_element_schur"));
  MH_CHECK(halo_u_exchange(s, u, nullptr));
  MH_CHECK(launch_element_mb(s, u));
  MH_CHECK(halo_v_exchange(s));
  return launch_face_reduce(s, u, w, 0, 0);
}

extern "C" int mh_get_element_schur(mh_system* s, int64_t first, int64_t count, double* out) {
  MH_CHECK(ready(s));
  MH_CHECK(need(s, s->have_mb, "element Schur blocks not formed"));
  if (first < 0 || count < 0 || first + count > s->N || (count && !out)) {
    set_error("macro range out of bounds");
    return MH_E_ARG;
  }
  const size_t blk = (size_t)s->nc * s->nc;
  if (count)
    MH_CHECK_CUDA(cudaMemcpy2DAsync(out, sizeof(double) * blk, s->S.p + first * s->ldS,
                                    sizeof(double) * (size_t)s->ldS, sizeof(double) * blk,
                                    (size_t)count, cudaMemcpyDeviceToHost, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  // stored transposed as +C A^-1 B; the reference's explicit block is
  // -(C A^-1 B) in row-major order
  const int nc = s->nc;
  std::vector<double> tmp(blk);
  for (int64_t b = 0; b < count; ++b) {
    double* o = out + b * blk;
    std::memcpy(tmp.data(), o, blk * sizeof(double));
    for (int r = 0; r < nc; ++r)
      for (int c = 0; c < nc; ++c) o[(size_t)r * nc + c] = -tmp[(size_t)c * nc + r];
  }
  return MH_OK;
}
