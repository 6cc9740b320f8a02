// Structured macro-mesh skeleton and condense tables (host C++).
//
// Replaces the connectivity half of the reference mesh builder
// (/root/reference/pkg/src/mehdg/mesh.py):
//   - 2-D macro enumeration, build_structured_macro_mesh (mesh.py:376-387):
//     cells row-major (j outer, i inner), triangles [p00,p10,p11], [p00,p11,p01];
//   - vertex ids by first visit (_dedup_vertices, mesh.py:331-345);
//   - local face k opposite vertex k, EDGE_VERTS (mesh.py:68);
//   - matching on the snapped vertex set, left side = lower macro id (mesh.py:232-245),
//     boundary faces on the square (mesh.py:247-258);
//   - face ids = lexicographic order of the canonical vertex tuple (mesh.py:304).
//     On the lattice x = i/n the 12-digit snap (_key, mesh.py:28-29) orders
//     exactly like the integer lattice coordinates, which we sort on.
//   - 3-D tets as _build_kuhn_counting_mesh (mesh.py:392-425); the 3-D skeleton
//     generalises the 2-D rules (the reference has none, mesh.py:372-375).
// Instead of the reference's dict of float tuples we sort 128-bit packed
// lattice keys, O(R log R) for R = (d+1) N face records.

#include <algorithm>
#include <array>
#include <cstring>
#include <numeric>
#include <vector>

#include "mh_internal.h"

namespace {

typedef unsigned __int128 u128;
constexpr int kBits = 12;  // lattice coordinate bits: n <= 4095

struct Rec {
  u128 key;
  int32_t elem;
  int32_t local;
};

int check_dim(int dim, int n) {
  if (dim != 2 && dim != 3) {
    mh::set_error("unsupported dimension (2 or 3)");
    return MH_E_ARG;
  }
  if (n < 1 || n >= (1 << kBits) - 1) {
    mh::set_error("n must satisfy 1 <= n < 4095");
    return MH_E_ARG;
  }
  return MH_OK;
}

// lattice points of macro e, in the reference's vertex order
void macro_points(int dim, int n, int64_t e, int pts[4][3]) {
  if (dim == 2) {
    int64_t cell = e / 2;
    int j = (int)(cell / n), i = (int)(cell % n);
    int p00[3] = {i, j, 0}, p10[3] = {i + 1, j, 0}, p11[3] = {i + 1, j + 1, 0},
        p01[3] = {i, j + 1, 0};
    const int* tri0[3] = {p00, p10, p11};
    const int* tri1[3] = {p00, p11, p01};
    const int** tri = (e % 2 == 0) ? tri0 : tri1;
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) pts[a][c] = tri[a][c];
  } else {
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                    {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    int64_t cube = e / 6;
    int pi = (int)(e % 6);
    int k = (int)(cube % n);
    int j = (int)((cube / n) % n);
    int i = (int)(cube / ((int64_t)n * n));
    int cur[3] = {i, j, k};
    for (int c = 0; c < 3; ++c) pts[0][c] = cur[c];
    for (int s = 0; s < 3; ++s) {
      cur[perms[pi][s]] += 1;
      for (int c = 0; c < 3; ++c) pts[s + 1][c] = cur[c];
    }
  }
}

bool lex_less(const int* a, const int* b, int dim) {
  for (int c = 0; c < dim; ++c)
    if (a[c] != b[c]) return a[c] < b[c];
  return false;
}

// face k of macro: vertex indices into the macro's point list
void face_vertices(int dim, int k, int idx[3]) {
  static const int edge[3][2] = {{1, 2}, {2, 0}, {0, 1}};  // mesh.py:68
  if (dim == 2) {
    idx[0] = edge[k][0];
    idx[1] = edge[k][1];
  } else {
    int q = 0;
    for (int a = 0; a < 4; ++a)
      if (a != k) idx[q++] = a;
  }
}

}  // namespace

extern "C" int mh_skeleton_sizes(int dim, int n, int64_t* n_elem, int64_t* n_vert,
                                 int64_t* n_face) {
  MH_CHECK(check_dim(dim, n));
  int64_t nn = n;
  if (dim == 2) {
    if (n_elem) *n_elem = 2 * nn * nn;
    if (n_vert) *n_vert = (nn + 1) * (nn + 1);
    if (n_face) *n_face = 3 * nn * nn + 2 * nn;  // (3n^2-2n) interior + 4n boundary
  } else {
    if (n_elem) *n_elem = 6 * nn * nn * nn;
    if (n_vert) *n_vert = (nn + 1) * (nn + 1) * (nn + 1);
    // interior 12n^3-6n^2 (costmodel.py:53) + boundary 12 n^2
    if (n_face) *n_face = 12 * nn * nn * nn + 6 * nn * nn;
  }
  return MH_OK;
}

extern "C" int mh_build_skeleton(int dim, int n, int32_t* verts, int32_t* elem_verts,
                                 int32_t* face_verts, int32_t* face_left,
                                 int32_t* face_right, int8_t* face_boundary,
                                 int32_t* elem_face) {
  MH_CHECK(check_dim(dim, n));
  int64_t N, NV, NF;
  mh_skeleton_sizes(dim, n, &N, &NV, &NF);
  const int nfe = dim + 1;
  const int64_t side = n + 1;
  std::vector<int32_t> vid((size_t)NV, -1);
  std::vector<std::array<int, 3>> coords;
  coords.reserve((size_t)NV);
  std::vector<int32_t> ev((size_t)(N * nfe));

  auto lattice_index = [&](const int* p) -> int64_t {
    return dim == 2 ? (int64_t)p[1] * side + p[0]
                    : ((int64_t)p[0] * side + p[1]) * side + p[2];
  };
  for (int64_t e = 0; e < N; ++e) {
    int pts[4][3];
    macro_points(dim, n, e, pts);
    for (int a = 0; a < nfe; ++a) {
      int64_t li = lattice_index(pts[a]);
      if (vid[li] < 0) {
        vid[li] = (int32_t)coords.size();
        coords.push_back({pts[a][0], pts[a][1], pts[a][2]});
      }
      ev[e * nfe + a] = vid[li];
    }
  }
  if ((int64_t)coords.size() != NV) {
    mh::set_error("vertex count mismatch");
    return MH_E_ARG;
  }

  std::vector<Rec> recs((size_t)(N * nfe));
  for (int64_t e = 0; e < N; ++e) {
    int pts[4][3];
    macro_points(dim, n, e, pts);
    for (int k = 0; k < nfe; ++k) {
      int idx[3];
      face_vertices(dim, k, idx);
      const int* fp[3];
      for (int q = 0; q < dim; ++q) fp[q] = pts[idx[q]];
      std::sort(fp, fp + dim, [&](const int* a, const int* b) { return lex_less(a, b, dim); });
      u128 key = 0;
      for (int q = 0; q < dim; ++q)
        for (int c = 0; c < dim; ++c) key = (key << kBits) | (u128)(unsigned)fp[q][c];
      recs[e * nfe + k] = Rec{key, (int32_t)e, (int32_t)k};
    }
  }
  std::sort(recs.begin(), recs.end(), [](const Rec& a, const Rec& b) {
    if (a.key != b.key) return a.key < b.key;
    return a.elem < b.elem;  // left = lower macro id (mesh.py:235)
  });

  int64_t fid = 0;
  size_t r = 0;
  while (r < recs.size()) {
    size_t g = r + 1;
    while (g < recs.size() && recs[g].key == recs[r].key) ++g;
    size_t cnt = g - r;
    if (cnt > 2) {
      mh::set_error("more than two macros share a face");
      return MH_E_ARG;
    }
    if (fid >= NF) {
      mh::set_error("face count mismatch");
      return MH_E_ARG;
    }
    const Rec& L = recs[r];
    // canonical vertices: decode the key back to lattice points
    int fpts[3][3] = {{0}};
    u128 key = L.key;
    for (int q = dim - 1; q >= 0; --q)
      for (int c = dim - 1; c >= 0; --c) {
        fpts[q][c] = (int)(unsigned)(key & (u128)((1u << kBits) - 1));
        key >>= kBits;
      }
    bool boundary = false;
    if (cnt == 1) {
      for (int c = 0; c < dim && !boundary; ++c)
        for (int v : {0, n}) {
          bool all = true;
          for (int q = 0; q < dim; ++q) all = all && fpts[q][c] == v;
          if (all) boundary = true;
        }
      if (!boundary) {
        mh::set_error("unmatched interior face");
        return MH_E_ARG;
      }
    }
    if (face_verts)
      for (int q = 0; q < dim; ++q) face_verts[fid * dim + q] = vid[lattice_index(fpts[q])];
    if (face_left) {
      face_left[fid * 2] = L.elem;
      face_left[fid * 2 + 1] = L.local;
    }
    if (face_right) {
      face_right[fid * 2] = cnt == 2 ? recs[r + 1].elem : -1;
      face_right[fid * 2 + 1] = cnt == 2 ? recs[r + 1].local : -1;
    }
    if (face_boundary) face_boundary[fid] = boundary ? 1 : 0;
    if (elem_face) {
      elem_face[(int64_t)L.elem * nfe + L.local] = (int32_t)fid;
      if (cnt == 2) elem_face[(int64_t)recs[r + 1].elem * nfe + recs[r + 1].local] = (int32_t)fid;
    }
    ++fid;
    r = g;
  }
  if (fid != NF) {
    mh::set_error("face count mismatch");
    return MH_E_ARG;
  }
  if (verts)
    for (int64_t v = 0; v < NV; ++v)
      for (int c = 0; c < dim; ++c) verts[v * dim + c] = coords[v][c];
  if (elem_verts) std::memcpy(elem_verts, ev.data(), ev.size() * sizeof(int32_t));
  return MH_OK;
}

extern "C" int mh_condense_tables(int nfe, int64_t n_elem, int64_t n_face_all,
                                  const int8_t* face_unknown, const int32_t* elem_face,
                                  const int32_t* face_left, const int32_t* face_right,
                                  int32_t* uidx, int32_t* elem_ufac, int32_t* face_elem,
                                  int32_t* face_slot, int64_t* n_unknown) {
  if (nfe < 1 || n_elem < 0 || n_face_all < 0 || !face_unknown || !elem_face || !face_left ||
      !face_right) {
    mh::set_error("mh_condense_tables: bad arguments");
    return MH_E_ARG;
  }
  std::vector<int32_t> u((size_t)n_face_all, -1);
  int64_t F = 0;
  for (int64_t f = 0; f < n_face_all; ++f)  // skeleton order, skip "D" (schur_solver.py:198-206)
    if (face_unknown[f]) u[f] = (int32_t)F++;
  if (uidx) std::memcpy(uidx, u.data(), u.size() * sizeof(int32_t));
  if (elem_ufac)
    for (int64_t i = 0; i < n_elem * nfe; ++i) {
      int32_t f = elem_face[i];
      if (f < -1 || f >= n_face_all) {
        mh::set_error("elem_face out of range");
        return MH_E_ARG;
      }
      elem_ufac[i] = f >= 0 ? u[f] : -1;
    }
  for (int64_t f = 0; f < n_face_all; ++f) {  // left then right (schur_solver.py:225-241)
    int32_t k = u[f];
    if (k < 0) continue;
    if (face_elem) {
      face_elem[2 * k] = face_left[2 * f];
      face_elem[2 * k + 1] = face_right[2 * f];
    }
    if (face_slot) {
      face_slot[2 * k] = face_left[2 * f + 1];
      face_slot[2 * k + 1] = face_right[2 * f + 1];
    }
  }
  if (n_unknown) *n_unknown = F;
  return MH_OK;
}

extern "C" int mh_slab_partition(int64_t n_elem, int64_t elems_per_slab, int nranks,
                                 int64_t* elem_begin) {
  if (nranks < 1 || n_elem < 0 || !elem_begin || elems_per_slab < 0) {
    mh::set_error("mh_slab_partition: bad arguments");
    return MH_E_ARG;
  }
  // whole slabs when the slab count divides into ranks as evenly as possible;
  // slab-less meshes (elems_per_slab == 0) cut the id range evenly.
  if (elems_per_slab > 0 && n_elem % elems_per_slab == 0 && n_elem / elems_per_slab >= nranks) {
    int64_t slabs = n_elem / elems_per_slab;
    for (int r = 0; r <= nranks; ++r) elem_begin[r] = (slabs * r / nranks) * elems_per_slab;
  } else {
    for (int r = 0; r <= nranks; ++r) elem_begin[r] = n_elem * r / nranks;
  }
  return MH_OK;
}
