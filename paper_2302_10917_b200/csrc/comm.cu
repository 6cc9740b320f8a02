// Multi-GPU halo exchange (NCCL over NVLink).  Single-device systems take
// the no-op path; the NCCL path is filled in by mh_set_halo / mh_comm_init.

#include "mh_internal.h"

namespace mh {

int halo_u_exchange(mh_system* s, const double* u, const double** u_halo) {
  (void)u;
  if (u_halo) *u_halo = s->halo_u.p;
  if (s->nranks <= 1) return MH_OK;
  set_error("multi-GPU halo exchange not initialised");
  return MH_E_STATE;
}

int halo_v_exchange(mh_system* s) {
  if (s->nranks <= 1) return MH_OK;
  set_error("multi-GPU halo exchange not initialised");
  return MH_E_STATE;
}

int halo_rhs_begin(mh_system* s) {
  (void)s;
  return MH_OK;
}

void free_comm(mh_system* s) { (void)s; }

}  // namespace mh

using namespace mh;

extern "C" int mh_set_halo(mh_system* s, int nranks, int rank, const int32_t* send_face,
                           const int32_t* send_count, const int32_t* recv_count,
                           const int32_t* vret_slot, const int32_t* vret_count,
                           const int32_t* vrecv_face, const int32_t* vrecv_count) {
  (void)s; (void)nranks; (void)rank; (void)send_face; (void)send_count; (void)recv_count;
  (void)vret_slot; (void)vret_count; (void)vrecv_face; (void)vrecv_count;
  set_error("multi-GPU halo not implemented yet");
  return MH_E_UNSUPPORTED;
}

extern "C" int mh_comm_unique_id(void* id_out_128) {
  (void)id_out_128;
  set_error("NCCL communicator not implemented yet");
  return MH_E_UNSUPPORTED;
}

extern "C" int mh_comm_init(mh_system* s, const void* id_128, int nranks, int rank) {
  (void)s; (void)id_128; (void)nranks; (void)rank;
  set_error("NCCL communicator not implemented yet");
  return MH_E_UNSUPPORTED;
}
