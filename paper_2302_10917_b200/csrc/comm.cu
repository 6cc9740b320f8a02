// Multi-GPU halo exchange and Krylov reductions over NCCL (NVLink 5 /
// NVSwitch).  NCCL is loaded at run time (dlopen of libnccl.so.2) so that
// the library shares whichever NCCL the process already uses (torch's).
//
// Messages per apply: the uhat halo owner -> neighbour,
// the v-slot contributions neighbour -> owner, and in GMRES one 8-byte
// all-gather per dot product.  Single-device systems take the no-op path.

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "mh_internal.h"

namespace mh {
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

int load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return MH_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    return MH_E_UNSUPPORTED;
  }
#define MH_SYM(field, name)                                               \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) {                                                    \
    set_error("libnccl is missing " name);                                \
    return MH_E_UNSUPPORTED;                                              \
  }
  MH_SYM(GetUniqueId, "ncclGetUniqueId")
  MH_SYM(CommInitRank, "ncclCommInitRank")
  MH_SYM(CommDestroy, "ncclCommDestroy")
  MH_SYM(GroupStart, "ncclGroupStart")
  MH_SYM(GroupEnd, "ncclGroupEnd")
  MH_SYM(Send, "ncclSend")
  MH_SYM(Recv, "ncclRecv")
  MH_SYM(AllGather, "ncclAllGather")
  MH_SYM(GetErrorString, "ncclGetErrorString")
#undef MH_SYM
  g_nccl.h = h;
  return MH_OK;
}

#define MH_CHECK_NCCL(expr)                                                        \
  do {                                                                             \
    ncclResult_t _r = (expr);                                                      \
    if (_r != ncclSuccess) {                                                       \
      ::mh::set_error(std::string(#expr) + ": " + g_nccl.GetErrorString(_r));     \
      return MH_E_CUDA;                                                            \
    }                                                                              \
  } while (0)

// out[i*t + s] = in[idx[i]*t + s]
__global__ void gather_segments(const double* __restrict__ in, const int32_t* __restrict__ idx,
                                int64_t count, int t, double* __restrict__ out) {
  const int64_t n = count * t;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / t;
    const int s = (int)(k - i * t);
    out[k] = in[(int64_t)idx[i] * t + s];
  }
}

__global__ void ordered_sum(const double* __restrict__ parts, int n, bool take_sqrt,
                            double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += parts[r];
    *out = take_sqrt ? sqrt(s) : s;
  }
}

int launch_gather(cudaStream_t st, const double* in, const int32_t* idx, int64_t count, int t,
                  double* out) {
  if (count <= 0) return MH_OK;
  const int64_t n = count * t;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
  gather_segments<<<grid, 256, 0, st>>>(in, idx, count, t, out);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

// grouped point-to-point exchange: send segments of sendbuf / receive into recvbuf
int exchange(mh_system* s, const double* sendbuf, const std::vector<int32_t>& scount,
             double* recvbuf, const std::vector<int32_t>& rcount) {
  ncclComm_t comm = (ncclComm_t)s->nccl;
  const int t = s->t;
  MH_CHECK_NCCL(g_nccl.GroupStart());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < s->nranks; ++q) {
    if (scount[q] > 0)
      MH_CHECK_NCCL(g_nccl.Send(sendbuf + so * t, (size_t)scount[q] * t, ncclFloat64, q, comm,
                                s->stream));
    if (rcount[q] > 0)
      MH_CHECK_NCCL(g_nccl.Recv(recvbuf + ro * t, (size_t)rcount[q] * t, ncclFloat64, q, comm,
                                s->stream));
    so += scount[q];
    ro += rcount[q];
  }
  MH_CHECK_NCCL(g_nccl.GroupEnd());
  return MH_OK;
}

bool multi(mh_system* s) { return multi_rank(s); }

int need_comm(mh_system* s) {
  if (!s->have_halo || !s->nccl) {
    set_error("multi-GPU system without halo plan / communicator");
    return MH_E_STATE;
  }
  return MH_OK;
}

}  // namespace

int halo_u_exchange(mh_system* s, const double* u, const double** u_halo) {
  if (u_halo) *u_halo = s->halo_u.p;
  if (!multi(s)) return MH_OK;
  MH_CHECK(need_comm(s));
  MH_CHECK(launch_gather(s->stream, u, s->send_face.p, (int64_t)s->send_face.n, s->t,
                         s->sendbuf.p));
  return exchange(s, s->sendbuf.p, s->send_count, s->halo_u.p, s->recv_count);
}

int halo_v_exchange(mh_system* s) {
  if (!multi(s)) return MH_OK;
  MH_CHECK(need_comm(s));
  MH_CHECK(launch_gather(s->stream, s->V.p, s->vret_slot.p, (int64_t)s->vret_slot.n, s->t,
                         s->vsendbuf.p));
  double* extra = s->V.p + (size_t)s->N * s->nfe * s->t;
  return exchange(s, s->vsendbuf.p, s->vret_count, extra, s->vrecv_count);
}

int halo_rhs_begin(mh_system* s) {
  (void)s;
  return MH_OK;
}

// m values per rank summed over ranks in rank order (identically on every rank)
__global__ void ordered_sum_vec(const double* __restrict__ parts, int nranks, int m,
                                double* __restrict__ out) {
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += parts[(size_t)r * m + i];
    out[i] = s;
  }
}

int allreduce_vec(mh_system* s, const double* local, int m, double* out) {
  if (!multi(s)) {
    ordered_sum_vec<<<1, 128, 0, s->stream>>>(local, 1, m, out);
    MH_CHECK_CUDA(cudaGetLastError());
    return MH_OK;
  }
  MH_CHECK(need_comm(s));
  MH_CHECK(s->dot_all.ensure((size_t)s->nranks * m));
  MH_CHECK_NCCL(g_nccl.AllGather(local, s->dot_all.p, (size_t)m, ncclFloat64,
                                 (ncclComm_t)s->nccl, s->stream));
  ordered_sum_vec<<<1, 128, 0, s->stream>>>(s->dot_all.p, s->nranks, m, out);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

int allreduce_scalar(mh_system* s, const double* local, double* out, bool take_sqrt) {
  if (!multi(s)) {
    ordered_sum<<<1, 32, 0, s->stream>>>(local, 1, take_sqrt, out);
    MH_CHECK_CUDA(cudaGetLastError());
    return MH_OK;
  }
  MH_CHECK(need_comm(s));
  MH_CHECK(s->dot_all.ensure((size_t)s->nranks));
  MH_CHECK_NCCL(g_nccl.AllGather(local, s->dot_all.p, 1, ncclFloat64, (ncclComm_t)s->nccl,
                                 s->stream));
  ordered_sum<<<1, 32, 0, s->stream>>>(s->dot_all.p, s->nranks, take_sqrt, out);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

void free_comm(mh_system* s) {
  s->send_face.release();
  s->vret_slot.release();
  s->sendbuf.release();
  s->vsendbuf.release();
  s->dot_local.release();
  s->dot_all.release();
  if (s->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)s->nccl);
  s->nccl = nullptr;
}

}  // namespace mh

using namespace mh;

extern "C" int mh_set_halo(mh_system* s, int nranks, int rank, const int32_t* send_face,
                           const int32_t* send_count, const int32_t* recv_count,
                           const int32_t* vret_slot, const int32_t* vret_count,
                           const int32_t* vrecv_count) {
  if (!s || nranks < 1 || rank < 0 || rank >= nranks || !send_count || !recv_count ||
      !vret_count || !vrecv_count) {
    set_error("mh_set_halo: bad arguments");
    return MH_E_ARG;
  }
  if (s->have_conn) {
    set_error("mh_set_halo must precede mh_upload_connectivity");
    return MH_E_STATE;
  }
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  s->nranks = nranks;
  s->rank = rank;
  s->send_count.assign(send_count, send_count + nranks);
  s->recv_count.assign(recv_count, recv_count + nranks);
  s->vret_count.assign(vret_count, vret_count + nranks);
  s->vrecv_count.assign(vrecv_count, vrecv_count + nranks);
  int64_t ns = 0, nr = 0, nv = 0, nvr = 0;
  for (int q = 0; q < nranks; ++q) {
    if (send_count[q] < 0 || recv_count[q] < 0 || vret_count[q] < 0 || vrecv_count[q] < 0 ||
        (q == rank && (send_count[q] || recv_count[q] || vret_count[q] || vrecv_count[q]))) {
      set_error("mh_set_halo: bad per-peer counts");
      return MH_E_ARG;
    }
    ns += send_count[q];
    nr += recv_count[q];
    nv += vret_count[q];
    nvr += vrecv_count[q];
  }
  for (int64_t i = 0; i < ns; ++i)
    if (send_face[i] < 0 || send_face[i] >= s->F) {
      set_error("mh_set_halo: send_face out of range");
      return MH_E_ARG;
    }
  for (int64_t i = 0; i < nv; ++i)
    if (vret_slot[i] < 0 || vret_slot[i] >= s->N * s->nfe) {
      set_error("mh_set_halo: vret_slot out of range");
      return MH_E_ARG;
    }
  s->F_halo = nr;
  s->n_vslot_extra = nvr;
  MH_CHECK(s->send_face.alloc((size_t)ns));
  MH_CHECK(s->vret_slot.alloc((size_t)nv));
  MH_CHECK(s->sendbuf.alloc((size_t)std::max<int64_t>(ns, 1) * s->t));
  MH_CHECK(s->vsendbuf.alloc((size_t)std::max<int64_t>(nv, 1) * s->t));
  MH_CHECK(s->halo_u.alloc((size_t)std::max<int64_t>(nr, 1) * s->t));
  if (ns)
    MH_CHECK_CUDA(cudaMemcpy(s->send_face.p, send_face, sizeof(int32_t) * ns,
                             cudaMemcpyHostToDevice));
  if (nv)
    MH_CHECK_CUDA(cudaMemcpy(s->vret_slot.p, vret_slot, sizeof(int32_t) * nv,
                             cudaMemcpyHostToDevice));
  s->have_halo = true;
  return MH_OK;
}

namespace {
// copy the segments q -> r of a grouped exchange (per-peer counts on both sides)
int group_exchange(mh_system** sys, int n, bool v_phase) {
  for (int r = 0; r < n; ++r) {
    mh_system* R = sys[r];
    int64_t ro = 0;
    for (int q = 0; q < n; ++q) {
      const int32_t cnt = v_phase ? R->vrecv_count[q] : R->recv_count[q];
      if (cnt > 0) {
        mh_system* S = sys[q];
        int64_t so = 0;  // offset of the q -> r block in q's send buffer
        for (int k = 0; k < r; ++k) so += v_phase ? S->vret_count[k] : S->send_count[k];
        const int32_t scnt = v_phase ? S->vret_count[r] : S->send_count[r];
        if (scnt != cnt) {
          set_error("group exchange: send/recv counts disagree");
          return MH_E_ARG;
        }
        const double* src = (v_phase ? S->vsendbuf.p : S->sendbuf.p) + so * S->t;
        double* dst = v_phase ? R->V.p + ((size_t)R->N * R->nfe + ro) * R->t
                              : R->halo_u.p + ro * R->t;
        MH_CHECK_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * cnt * R->t,
                                      cudaMemcpyDeviceToDevice, R->stream));
      }
      ro += cnt;
    }
  }
  return MH_OK;
}
}  // namespace

extern "C" int mh_group_apply(mh_system** sys, int n, const double** u, double** w) {
  if (!sys || n < 1 || !u || !w) return MH_E_ARG;
  for (int r = 0; r < n; ++r)
    if (!sys[r] || !sys[r]->factored || !sys[r]->have_halo || sys[r]->nranks != n ||
        sys[r]->rank != r) {
      set_error("mh_group_apply: every system needs a halo plan for rank r of n and factors");
      return MH_E_STATE;
    }
  // all systems must see each other's buffers in stream order: run on one stream
  for (int r = 0; r < n; ++r) MH_CHECK_CUDA(cudaStreamSynchronize(sys[r]->stream));
  for (int r = 0; r < n; ++r)
    MH_CHECK(launch_gather(sys[r]->stream, u[r], sys[r]->send_face.p,
                           (int64_t)sys[r]->send_face.n, sys[r]->t, sys[r]->sendbuf.p));
  for (int r = 0; r < n; ++r) MH_CHECK_CUDA(cudaStreamSynchronize(sys[r]->stream));
  MH_CHECK(group_exchange(sys, n, false));
  for (int r = 0; r < n; ++r) {
    MH_CHECK(launch_element(sys[r], kApply, u[r], sys[r]->V.p));
    MH_CHECK(launch_gather(sys[r]->stream, sys[r]->V.p, sys[r]->vret_slot.p,
                           (int64_t)sys[r]->vret_slot.n, sys[r]->t, sys[r]->vsendbuf.p));
  }
  for (int r = 0; r < n; ++r) MH_CHECK_CUDA(cudaStreamSynchronize(sys[r]->stream));
  MH_CHECK(group_exchange(sys, n, true));
  for (int r = 0; r < n; ++r) MH_CHECK(launch_face_reduce(sys[r], u[r], w[r], 0, 0));
  for (int r = 0; r < n; ++r) MH_CHECK_CUDA(cudaStreamSynchronize(sys[r]->stream));
  return MH_OK;
}

extern "C" int mh_comm_unique_id(void* id_out) {
  if (!id_out) return MH_E_ARG;
  MH_CHECK(load_nccl());
  ncclUniqueId id;
  MH_CHECK_NCCL(g_nccl.GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return MH_OK;
}

extern "C" int mh_comm_init(mh_system* s, const void* id_in, int nranks, int rank) {
  if (!s || !id_in || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("mh_comm_init: bad arguments");
    return MH_E_ARG;
  }
  MH_CHECK(load_nccl());
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof(id));
  ncclComm_t comm = nullptr;
  MH_CHECK_NCCL(g_nccl.CommInitRank(&comm, nranks, id, rank));
  s->nccl = comm;
  s->nranks = nranks;
  s->rank = rank;
  return MH_OK;
}
