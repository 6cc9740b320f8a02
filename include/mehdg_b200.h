/*
 * mehdg_b200.h -- C-ABI of the B200-native macro-element Schur-operator path.
 *
 * The reference (arxiv 2302.10917, package `mehdg`) is pure Python; its
 * hot path sits behind the Python API of `mehdg.schur_solver`
 * (/root/reference/pkg/src/mehdg/schur_solver.py).  It has no FFI of its
 * own, so each entry point below names the reference function it replaces;
 * INTEGRATION.md shows the ctypes binding a maintainer would add.
 *
 * Conventions
 *   - every call returns MH_OK (0) or a negative MH_E* status code;
 *     mh_last_error() returns a static message for the calling thread;
 *   - plain pointers and sizes only; "_host" pointers are host memory,
 *     "_dev" pointers are device memory on the system's device;
 *   - all device work is enqueued on the system's stream (mh_set_stream);
 *     calls that return host data synchronise that stream;
 *   - block layouts are the reference's (row-major numpy C order):
 *       A    N x Q x Q        op.A                 (assembly.py:63-72)
 *       B    N x Q x nc       op.B  (BASELINE B_e^T)
 *       C    N x nc x Q       op.C  (BASELINE B_e)
 *       R_u  N x Q
 *       D    F x t x t        FaceOperator.D of the F unknown faces (assembly.py:75-82)
 *       R_hat F x t
 *     Trace vectors (uhat, w, f) are zhat = F*t long, face-contiguous in
 *     unknown-face order (the `offsets` of condense, schur_solver.py:198-206).
 */
#ifndef MEHDG_B200_H
#define MEHDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------- */
#define MH_OK 0
#define MH_E_ARG (-1)          /* invalid argument (ValueError in the reference)      */
#define MH_E_CUDA (-2)         /* CUDA runtime failure                                 */
#define MH_E_NOMEM (-3)        /* device allocation failed                             */
#define MH_E_SINGULAR_LOCAL (-4) /* SingularLocalBlock(macro_id), schur_solver.py:33   */
#define MH_E_SINGULAR_FACE (-5)  /* SingularFaceBlock(face_id),  schur_solver.py:37    */
#define MH_E_STATE (-6)        /* call out of order (e.g. apply before factorize)      */
#define MH_E_UNSUPPORTED (-7)  /* shape outside what the kernels support               */
#define MH_E_CALLBACK (-8)     /* a user operator callback returned non-zero           */

/* face factor kinds, FaceOperator.factor_kind (schur_solver.py:130-147) */
#define MH_FACE_CHOL_NEG 0
#define MH_FACE_CHOL_POS 1
#define MH_FACE_LU 2
#define MH_FACE_SINGULAR (-1)

typedef struct mh_system mh_system; /* opaque; one condensed system on one device */

const char* mh_last_error(void);
int mh_version(void);
/* Number of CUDA devices visible; 0 on a host without a GPU (no error). */
int mh_device_count(int* count);

/* ---- connectivity (host code; replaces build_structured_macro_mesh's
 *      skeleton, mesh.py:207-321 / 359-425) ------------------------------ */

/* Sizes of the structured macro mesh of [0,1]^dim (dim 2 or 3). */
int mh_skeleton_sizes(int dim, int n, int64_t* n_elem, int64_t* n_vert, int64_t* n_face);

/* Skeleton tables (integer-exact with the reference 2-D skeleton):
 *   verts[n_vert*dim]        lattice coordinates (x = i/n)
 *   elem_verts[n_elem*(dim+1)]
 *   face_verts[n_face*dim]   vertex ids in canonical (sorted) order
 *   face_left[n_face*2]      (macro, local face) of the lower-id side
 *   face_right[n_face*2]     (macro, local face) or (-1,-1) on the boundary
 *   face_boundary[n_face]    1 on the domain boundary (tag "D" by default)
 *   elem_face[n_elem*(dim+1)] face id of local face k (opposite vertex k) */
int mh_build_skeleton(int dim, int n, int32_t* verts, int32_t* elem_verts,
                      int32_t* face_verts, int32_t* face_left, int32_t* face_right,
                      int8_t* face_boundary, int32_t* elem_face);

/* condense's integer tables (schur_solver.py:198-241) for uniform slot width:
 *   face_unknown[n_face_all]   1 for faces that carry unknowns (tag != "D")
 *   uidx[n_face_all]           unknown index or -1 (offsets start = uidx*t)
 *   elem_ufac[n_elem*nfe]      unknown index of local face k or -1 (gather table)
 *   face_elem[n_unknown*2], face_slot[n_unknown*2]  left-then-right plan
 * n_unknown receives the number of unknown faces F. */
int mh_condense_tables(int nfe, int64_t n_elem, int64_t n_face_all,
                       const int8_t* face_unknown, const int32_t* elem_face,
                       const int32_t* face_left, const int32_t* face_right,
                       int32_t* uidx, int32_t* elem_ufac, int32_t* face_elem,
                       int32_t* face_slot, int64_t* n_unknown);

/* Contiguous slab partition for multi-GPU runs: rank r owns macros
 * [elem_begin[r], elem_begin[r+1]) (whole mesh rows / x-slabs when they
 * divide evenly, else a cut of the id range) and every unknown face whose
 * left (lower-id) macro it owns. */
int mh_slab_partition(int64_t n_elem, int64_t elems_per_slab, int nranks, int64_t* elem_begin);

/* ---- system lifecycle (replaces condense, schur_solver.py:185-254) ---- */

/* Create a system of n_elem macros with Q x Q blocks, nfe face slots of width
 * t each (nc = nfe*t; nfe = dim+1 on conforming meshes, up to 6 on 2-D meshes
 * with hanging faces -- macros with fewer faces leave their last slots empty),
 * and n_face unknown faces, on device `device`. */
int mh_create(int device, int nfe, int64_t n_elem, int q, int t, int64_t n_face,
              mh_system** out);
int mh_destroy(mh_system* sys);
/* Use an external stream (e.g. torch.cuda.current_stream().cuda_stream). */
int mh_set_stream(mh_system* sys, void* stream);

/* Connectivity from mh_condense_tables (host arrays). */
int mh_upload_connectivity(mh_system* sys, const int32_t* elem_ufac_host,
                           const int32_t* face_elem_host, const int32_t* face_slot_host);

/* Blocks (host arrays, reference layouts above).  Either B or C may be NULL:
 * B == NULL means op.B = op.C^T, C == NULL means op.C = op.B^T (the
 * BASELINE synthetic operator, stored and streamed once).  R_u / R_hat may be
 * NULL (zeros). */
int mh_upload_blocks(mh_system* sys, const double* A_host, const double* B_host,
                     const double* C_host, const double* R_u_host,
                     const double* D_host, const double* R_hat_host);
/* Same, from device memory (no host staging). */
int mh_upload_blocks_device(mh_system* sys, const double* A_dev, const double* B_dev,
                            const double* C_dev, const double* R_u_dev,
                            const double* D_dev, const double* R_hat_dev);

/* _factorize_local for all macros + _factorize_face for all faces
 * (schur_solver.py:105-147).  On MH_E_SINGULAR_LOCAL / _FACE the lowest
 * failing macro / face index is returned in *fail_macro / *fail_face (-1
 * otherwise).  face_kinds_host (n_face int8, may be NULL) receives
 * MH_FACE_* per face.  Timing in ms of the LU kernel in *lu_ms (may be NULL). */
int mh_factorize(mh_system* sys, int32_t* fail_macro, int32_t* fail_face,
                 int8_t* face_kinds_host, float* lu_ms);
/* Re-run only the batched LU (benchmarking); A must still be staged. */
int mh_refactorize_local(mh_system* sys, float* lu_ms);

/* Factors in LAPACK layout for parity (scipy.linalg.lu_factor):
 * lu_host[n*Q*Q] row-major packed L\U, piv_host[n*Q] 0-based pivots,
 * for macros [first, first+count). */
int mh_get_local_factors(mh_system* sys, int64_t first, int64_t count,
                         double* lu_host, int32_t* piv_host);

/* The preconditioner's face inverses D_f^-1 (sign folded in) of the n
 * unknown faces idx[], t x t row-major on the host.  The set form replaces
 * them -- the drop-in honours a face factor replaced after condense
 * (the reference's op.factor, schur_solver.py:137-154, 296-305). */
int mh_get_face_inverse(mh_system* sys, int64_t n, const int32_t* idx, double* inv_host);
int mh_set_face_inverse(mh_system* sys, int64_t n, const int32_t* idx, const double* inv_host);

/* ---- the operator (device pointers, zhat doubles) -------------------- */

/* f = R_hat - sum_e C A^-1 R_u   (condense reduced RHS, schur_solver.py:243-253) */
int mh_rhs(mh_system* sys, double* f_dev);
/* w = (D - C A^-1 B) uhat        (apply_schur, schur_solver.py:267-293) */
int mh_apply(mh_system* sys, const double* uhat_dev, double* w_dev);
/* z = D^-1 w per face            (apply_preconditioner, schur_solver.py:296-305) */
int mh_precond(mh_system* sys, const double* w_dev, double* z_dev);
/* z = D^-1 (D - C A^-1 B) uhat  (the fused M(A v) GMRES step) */
int mh_apply_precond(mh_system* sys, const double* uhat_dev, double* z_dev);
/* U[n_elem*Q] = A^-1 (R_u - B gather(uhat))  (reconstruct_interior, :423-431) */
int mh_reconstruct(mh_system* sys, const double* uhat_dev, double* U_dev);
/* Host-buffer variants (copies inside, stream-synchronous). */
int mh_apply_host(mh_system* sys, const double* uhat_host, double* w_host);
int mh_precond_host(mh_system* sys, const double* w_host, double* z_host);
int mh_rhs_host(mh_system* sys, double* f_host);
int mh_reconstruct_host(mh_system* sys, const double* uhat_host, double* U_host);
/* w_i = (D - C A^-1 B) u_i for k host vectors u_i = uhat_host + i*ldu,
 * w_i = w_host + i*ldw (strides in doubles; 0 reuses one input / overwrites
 * one output).  The host->device copy of vector i+1 and the device->host copy
 * of vector i-1 overlap the apply of vector i (two copy streams, two device
 * buffer pairs); returns when every w_i is in host memory.  Pinned host memory
 * lets the copies run asynchronously. */
int mh_apply_host_many(mh_system* sys, int64_t k, const double* uhat_host, int64_t ldu,
                       double* w_host, int64_t ldw);

/* ---- device assembly of the 2-D HDG blocks (assembly.py:170-322) ----------
 * Reference-element tables (device pointers) of a conforming structured mesh,
 * built by paper_2302_10917_b200/fem.py; nloc = 3 Q, nc = 3 t. */
typedef struct {
  int32_t m, p, Q, nb, t, nq, ncell, nfq, nffq, supg, supg_plus;
  double kappa, ax, ay;
  const double* qw;         /* nq quadrature weights on the reference triangle */
  const double* val;        /* nq x nb basis values */
  const double* gref;       /* nq x nb x 2 reference gradients */
  const double* href;       /* nq x nb x 2 x 2 reference Hessians (SUPG) */
  const int32_t* cell_kind; /* ncell: 0 "up", 1 "down" (mesh.py:71-77 order) */
  const int32_t* cell_map;  /* ncell x nb sub-cell dof -> patch dof */
  const int32_t* edge_nodes;/* 3 x t patch dofs along each macro edge */
  const double* fw;         /* 6 x nfq weights of assemble_macro's face rule per side
                               variant (t0, t1) = (0,1) (1,0) (0,.5) (.5,0) (.5,1) (1,.5),
                               zero padded */
  const double* th;         /* 6 x nfq x t macro-edge trace basis at t0 + (t1 - t0) s */
  const double* ps;         /* 6 x nfq x t face trace basis at s */
  const double* ffw;        /* nffq weights of assemble_face's rule */
  const double* fps;        /* nffq x t */
} mh_hdg2d_tables;
/* assemble_macro for N macros with nslot face slots each (3, or up to 6 with
 * 2:1 hanging faces): verts[N*3*2]; per slot (N*nslot, in the macro's face
 * order): slot_edge (local edge, -1 = empty slot), slot_var (side variant),
 * slot_dirichlet (row of ghat[nD*t] for a Dirichlet face, else -1), slot_len
 * (face length); fq[N*ncell*nq] (f at the physical quadrature points).
 * Outputs (device, row-major, nc = nslot*t): A[N*nloc*nloc], B[N*nloc*nc]
 * (op.B), C[N*nc*nloc] (op.C), Ru[N*nloc].  stream: cudaStream_t. */
int mh_assemble_macros_2d(const mh_hdg2d_tables* tab, int64_t N, int nslot, const double* verts,
                          const int8_t* slot_edge, const int8_t* slot_var,
                          const int32_t* slot_dirichlet, const double* slot_len,
                          const double* ghat, const double* fq, double* A, double* B, double* C,
                          double* Ru, void* stream);
/* assemble_face's D block for F faces: face_sides[F*4] = (left macro, left
 * edge, right macro or -1, right edge), face_len[F]; D[F*t*t] row-major. */
int mh_assemble_faces_2d(const mh_hdg2d_tables* tab, int64_t F, const double* verts,
                         const int32_t* face_sides, const double* face_len, double* D,
                         void* stream);

/* ---- explicit (matrix-based) Schur, mode "mb" (schur_solver.py:388-420) */
/* Form S_e = C A^-1 B (nc x nc) per macro on the device; afterwards
 * mh_apply_mb computes w = D uhat - sum_e S_e uhat_e with the same face
 * reduction order as mh_apply. */
int mh_form_element_schur(mh_system* sys);
int mh_apply_mb(mh_system* sys, const double* uhat_dev, double* w_dev);
/* Download -S_e (the reference's explicit element blocks) for
 * macros [first, first+count): out_host[count*nc*nc] row-major. */
int mh_get_element_schur(mh_system* sys, int64_t first, int64_t count, double* out_host);

/* ---- per-kernel timing (CUDA events around each launch) ---------------- */
/* enable != 0 starts recording events around the element and face kernels
 * launched by the operator entry points; mh_profile_read synchronises the
 * stream, returns the summed durations (ms) and launch counts since the last
 * read, and clears them. */
int mh_profile(mh_system* sys, int enable);
int mh_profile_read(mh_system* sys, double* elem_ms, int64_t* elem_launches,
                    double* face_ms, int64_t* face_launches);

/* ---- GMRES (schur_solver.py:308-385) ----------------------------------- */

/* Operator callback: out_dev = Op(in_dev), both n doubles on the device. */
typedef int (*mh_op_fn)(void* ctx, const double* in_dev, double* out_dev);

/* Restarted, left-preconditioned GMRES with MGS and Givens rotations, the
 * reference's control flow and stopping rule.  x_dev receives the solution
 * (x0 = 0).  hist_host (hist_cap doubles) receives the residual history,
 * *hist_len its full length.  mode: 0 matrix-free, 1 matrix-based. */
int mh_gmres(mh_system* sys, double tol, int restart, int maxiter, int use_precond,
             int mode, const double* rhs_dev, double* x_dev, int* iterations,
             int* converged, double* hist_host, int hist_cap, int* hist_len);
/* Same algorithm for arbitrary operators (e.g. the reference's KATs);
 * precond may be NULL (identity).  stream may be NULL (legacy default). */
int mh_gmres_op(int device, void* stream, int64_t n, mh_op_fn apply, void* apply_ctx,
                mh_op_fn precond, void* precond_ctx, double tol, int restart,
                int maxiter, const double* rhs_dev, double* x_dev, int* iterations,
                int* converged, double* hist_host, int hist_cap, int* hist_len);

/* Deterministic fixed-partition dot product of device vectors (host result). */
int mh_dot(void* stream, int64_t n, const double* x_dev, const double* y_dev, double* out_host);

/* ---- multi-GPU (NCCL over NVLink) ------------------------------------- */
/* Slab decomposition: rank r owns macros
 * [elem_begin[r], elem_begin[r+1]) and the unknown faces whose left
 * (lower-id) macro it owns.  Its trace vector is [owned faces | halo faces];
 * halo faces (right macro here, left macro on rank q) are grouped by owner q
 * ascending, then by global face index.  Per apply:
 *   1. uhat halo: rank q sends the owned segments listed in send_face (grouped
 *      by destination, send_count[dest] each) and receives recv_count[src]
 *      contiguous halo segments from each source;
 *   2. element kernel on the local macros;
 *   3. v return: the slot segments listed in vret_slot (grouped by owner,
 *      vret_count[owner] each) go back to the face owners, which receive
 *      vrecv_count[src] contiguous segments into extra v-slots and subtract
 *      them second, i.e. in the reference's left-then-right order -- so the
 *      multi-GPU apply is bitwise identical to the single-GPU one.
 * Krylov dot products are all-gathered and summed in rank order.
 * mh_set_halo must precede mh_upload_connectivity; face_elem entries >= the
 * local macro count address received v-slot segments (N + j). */
int mh_set_halo(mh_system* sys, int nranks, int rank, const int32_t* send_face_host,
                const int32_t* send_count_host, const int32_t* recv_count_host,
                const int32_t* vret_slot_host, const int32_t* vret_count_host,
                const int32_t* vrecv_count_host);
/* Apply the operator of a slab-partitioned problem held by n systems in ONE
 * process (system r = rank r, halo plans set, no communicator): the same
 * pack / exchange / element / v-return / face phases as the NCCL path, with
 * the exchanges done by device-to-device copies.  Used to verify the halo
 * plans and kernels on a single GPU; u_dev[r] / w_dev[r] are rank-local. */
int mh_group_apply(mh_system** systems, int n, const double** u_dev, double** w_dev);
/* ncclUniqueId bytes (128); rank 0 creates it and the caller broadcasts it. */
int mh_comm_unique_id(void* id_out_128);
/* NCCL communicator over all ranks (libnccl.so.2 is loaded at run time). */
int mh_comm_init(mh_system* sys, const void* id_128, int nranks, int rank);

#ifdef __cplusplus
}
#endif
#endif /* MEHDG_B200_H */
