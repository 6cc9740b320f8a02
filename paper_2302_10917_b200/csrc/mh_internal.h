// Internal declarations shared by the translation units of libmehdg_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>
#include <utility>
#include <string>
#include <vector>

#include "../../include/mehdg_b200.h"

namespace mh {

void set_error(const std::string& msg);

#define MH_CHECK_CUDA(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::mh::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));     \
      return MH_E_CUDA;                                                       \
    }                                                                         \
  } while (0)

#define MH_CHECK(expr)        \
  do {                        \
    int _s = (expr);          \
    if (_s != MH_OK) return _s; \
  } while (0)

constexpr int kWarp = 32;
// face slots per macro: d + 1 on conforming meshes, up to 6 with 2:1 hanging
// faces in 2-D (two faces per macro edge, mesh.py:264-302)
constexpr int kMaxSlots = 6;
constexpr unsigned kFull = 0xffffffffu;
// fixed reduction partition: results never depend on the device or SM count
// chunk (doubles) of the element kernel's bulk-copy stream; the per-macro
// strides of the streamed arrays (op.B^T, L, U, op.C) are multiples of it
constexpr int kStreamChunk = 512;

// Device buffer with RAII-less explicit free (the system owns them).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    if (count == n && p) return MH_OK;
    release();
    if (count == 0) return MH_OK;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      set_error(std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
      return MH_E_NOMEM;
    }
    n = count;
    return MH_OK;
  }
  // grow-only: keeps a buffer that enqueued work may still use when it is large enough
  int ensure(size_t count) { return count <= n && p ? MH_OK : alloc(count); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct Krylov;  // GMRES workspace (krylov.cu)

// Tuning knobs: read from the environment once, when a
// system is created, never on a launch path.  Defaults are the measured best.
struct Knobs {
  int lu = 0;             // MEHDG_LU: 0 default (pipe where it fits), 1 tile, 2 cta, 3 pipe
  int lu_pipe_w = 0;      // MEHDG_LU_PIPE_W: warps per block of the pipelined LU (0: by size)
  int lu_pipe_ctas = 0;   // MEHDG_LU_PIPE_CTAS: cap on its CTAs per SM (0: none)
  int lu_ctas = 3;        // MEHDG_LU_CTAS: resident CTAs per SM of the tile LU
  int lu_scr_pol = 0;     // MEHDG_LU_SCR: L2 policy of the tile LU's scratch
  int lu_a_pol = 1;       // MEHDG_LU_APOL: L2 policy of the A stream (1 evict_first)
  int elem_ctas = 0;      // MEHDG_ELEM_CTAS: cap on element-kernel CTAs per SM (0: none)
  int elem_ch = 512;      // MEHDG_ELEM_CH: element stream chunk (doubles)
  int elem_bpol = 1;      // MEHDG_ELEM_BPOL: L2 policy of op.B^T's first read when it is re-read (0 evict_first, 1 evict_last, 2 normal, 3 half evict_last)
  int elem_split = 0;      // MEHDG_ELEM_SPLIT: apply-mode element kernel with a macro split over its row groups
  int elem_split_ctas = 0; // MEHDG_ELEM_SPLIT_CTAS: its CTAs (macros in flight) per SM (0: by L2 footprint)
  int mb_stream = 1;      // MEHDG_MB_STREAM: the mb apply through the element kernel's TMA stream
  int elem_lpol = 0;      // MEHDG_ELEM_LPOL: L2 policy of the L / U streams (0 evict_first, 2 normal)
  int mgs_small = 1;      // MEHDG_MGS_SMALL: the MGS block of a step as one kernel
  int mgs_ctas = 4;       // MEHDG_MGS_CTAS: its CTAs per SM (at most)
  int mgs_reg = 1;        // MEHDG_MGS_REG: w held in registers when it fits
  int face_bulk = 1;      // MEHDG_FACE_BULK: TMA-staged face kernel for t > 32
  int gmres_graphs = 1;   // MEHDG_GMRES_GRAPHS: MGS block as a CUDA graph
  int64_t split_at = -1;  // MEHDG_SPLIT_AT: interior/halo macro split (-1: computed)
  void read();
};

}  // namespace mh

struct mh_system {
  mh::Knobs knobs;
  int device = 0;
  int nfe = 3;        // faces (slots) per macro = d+1
  int64_t N = 0;      // macros on this device
  int Q = 0;          // block size
  int t = 0;          // trace dofs per face
  int nc = 0;         // slot dofs per macro = nfe*t
  int64_t F = 0;      // unknown faces owned (trace vector = F*t)
  int64_t F_halo = 0; // halo faces (multi-GPU); trace buffer = (F+F_halo)*t
  int64_t n_vslot_extra = 0;  // received v-slot segments (multi-GPU)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t cin = nullptr, cout = nullptr;  // copy streams of mh_apply_host_many
  cudaEvent_t evp[7] = {};
  bool have_conn = false, have_blocks = false, factored = false, have_mb = false;
  bool c_is_bt = false;
  int max_smem_optin = 0;
  int num_sms = 0;

  // connectivity
  mh::DBuf<int32_t> elem_ufac;   // N*nfe   unknown face (local trace index) or -1
  mh::DBuf<int32_t> face_vslot;  // F*2     v-slot index (e*nfe+k) left, right or -1
  // host copies of the tables (for halo planning / introspection)
  std::vector<int32_t> h_face_elem, h_face_slot;

  // blocks
  mh::DBuf<double> A;      // staged A, N*Q*Q row-major (input of the LU)
  mh::DBuf<double> lu_scr; // per-warp-slot scratch of the tile LU (inverse diagonal blocks)
  mh::DBuf<int64_t> lu_fb; // pipelined LU: [0] count, [1..] blocks handed to the tile kernel
  int lu_fallback_blocks = 0;  // how many the last factorisation handed over
  mh::DBuf<double> Lp;     // N*ldL packed strict lower L, columns 0..Q-2 (streamed)
  mh::DBuf<double> Up;     // N*ldL packed strict upper U, columns Q-1..1 (streamed)
  mh::DBuf<double> udiag;  // N*Q   diag(U)
  int64_t ldB = 0;         // per-macro stride of Bt / Cm (nc*Q rounded up to kStreamChunk)
  int64_t ldL = 0;         // per-macro stride of Lp / Up (Q(Q-1)/2 rounded up to kStreamChunk)
  int64_t ldS = 0;         // per-macro stride of S (nc*nc rounded up to kStreamChunk)
  int64_t ldF = 0;         // per-face stride of D / Dinv (t*t rounded up to 16 bytes)
  mh::DBuf<double> dinv;   // N*Q   1/U_ii
  mh::DBuf<int32_t> piv;   // N*Q   LAPACK 0-based pivots
  mh::DBuf<int32_t> perm;  // N*Q   composed row permutation: (P x)_i = x[perm_i]
  mh::DBuf<int32_t> lstat; // N     1 if singular
  mh::DBuf<double> Bt;     // N*nc*Q  op.B^T  (row c = column c of op.B)
  mh::DBuf<double> Cm;     // N*nc*Q  op.C    (aliases Bt when c_is_bt)
  mh::DBuf<double> Ru;     // N*Q
  mh::DBuf<double> D;      // F*ldF  column-major face blocks
  mh::DBuf<double> Draw;   // F*t*t  row-major face blocks as uploaded (factor input)
  mh::DBuf<double> Rhat;   // F*t
  mh::DBuf<double> Dinv;   // F*ldF  D_f^-1 column-major (sign folded in)
  mh::DBuf<int8_t> Fkind;  // F
  mh::DBuf<double> V;      // (N*nfe + extra)*t  element slot contributions
  mh::DBuf<double> tmp;    // F*t scratch
  mh::DBuf<double> S;      // N*nc*nc element Schur blocks (mode mb)
  mh::DBuf<double> halo_u; // received halo trace segments [F_halo*t] (multi-GPU)
  mh::DBuf<double> hin, hout;  // staging for the *_host entry points

  mh::Krylov* kry = nullptr;
  // set while a pipelined GMRES cycle runs: the element / face kernels of a
  // step enqueued after the cycle stopped return at once
  const int* skip = nullptr;

  // optional per-kernel event timing (mh_profile)
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_elem, ev_face;

  // multi-GPU (comm.cu)
  int nranks = 1, rank = 0;
  void* nccl = nullptr;  // ncclComm_t
  // macros [0, e_split) read received halo traces; [e_split, N) run on kstream
  // while the halo exchange is in flight (mh_apply on a multi-rank system)
  int64_t e_split = 0;
  cudaStream_t kstream = nullptr;
  cudaEvent_t ev_u = nullptr, ev_int = nullptr;
  bool have_halo = false;
  std::vector<int32_t> send_count, recv_count, vret_count, vrecv_count;  // per peer
  mh::DBuf<int32_t> send_face, vret_slot;
  mh::DBuf<double> sendbuf, vsendbuf;
  mh::DBuf<double> dot_local, dot_all;  // Krylov all-gather scratch
};

namespace mh {
// capi.cu: resident CTAs per SM of `kern` at (threads, smem); sets the
// function's max-dynamic-smem attribute (raise-only, process-wide cache);
// -1 (error set) on failure
int launch_occupancy(int device, const void* kern, int threads, size_t smem);
// lu.cu
int launch_lu(mh_system* s, float* ms);
// element.cu
enum ElemMode { kApply = 0, kRhs = 1, kRecon = 2, kMb = 3 };  // kMb: v = S_e ue (explicit element Schur)
int launch_element(mh_system* s, int mode, const double* uhat, double* out);
// a system with a communicator takes the NCCL path even with one rank (the
// single-GPU box's test of the NCCL calls); plain systems the no-op path
inline bool multi_rank(const mh_system* s) { return s->nranks > 1 || s->nccl != nullptr; }
// macros [e_lo, e_hi) on stream st
int launch_element_range(mh_system* s, int mode, const double* uhat, double* out,
                         cudaStream_t st, int64_t e_lo, int64_t e_hi);
int launch_element_schur(mh_system* s);
int launch_element_mb(mh_system* s, const double* uhat);
int launch_element_mb_stream(mh_system* s, const double* uhat, double* out);  // element.cu
// face.cu
int launch_face_factor(mh_system* s, const double* Drm);
int launch_face_reduce(mh_system* s, const double* uhat, double* w, int rhs_mode, int fuse_precond);
int launch_precond(mh_system* s, const double* w, double* z);
int launch_transpose_batched(cudaStream_t st, const double* in, double* out, int64_t batch,
                             int rows, int cols, int64_t out_stride = -1);
int launch_unpack_lu(mh_system* s, int64_t first, int64_t count, double* out_rowmajor);
// krylov.cu
void free_krylov(Krylov* k);
// capi.cu: event-timed launch brackets (no-ops unless profiling)
int prof_begin(mh_system* s, cudaEvent_t* ev);
int prof_end(mh_system* s, cudaEvent_t ev0, int kind);  // kind 0 element, 1 face
// comm.cu (multi-GPU halo; no-ops on a single device)
int halo_u_exchange(mh_system* s, const double* u, const double** u_halo);
int halo_v_exchange(mh_system* s);
int halo_rhs_begin(mh_system* s);
void free_comm(mh_system* s);
// sum a device scalar over ranks (rank order) into out; sqrt if requested
int allreduce_scalar(mh_system* s, const double* local, double* out, bool take_sqrt);
// m values per rank, each summed over ranks in rank order, into out[m] (device)
int allreduce_vec(mh_system* s, const double* local, int m, double* out);
}  // namespace mh
