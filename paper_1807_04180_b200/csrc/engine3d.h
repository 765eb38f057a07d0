// Host-side structures of the engine's 3-D path (BASELINE config 5). The math
// is the restatement oracle/hddm_oracle3.c (the reference has no 3-D code);
// the data layout is DESIGN.md section 10.
//
//  * every subdomain window has the same node counts, so ONE symbolic structure
//    (shell-first plane-separator ND order, supernode tree, dense supernode
//    row structures) serves every class;
//  * per-subdomain vectors are stored subdomain-major in factor order;
//  * global fields are x fastest, then y, then z.
#pragma once

#include <string>
#include <vector>

#include "hddm3.h"

namespace hddm3 {

// One nested-dissection supernode: a leaf box (natural order inside) or a
// separator plane eliminated after both halves. Its rows are the ancestor
// positions its subtree couples to (sorted ascending); its L is stored as
// dense blocks: the inverse of the unit-lower diagonal block (packed, column
// major, strictly lower) and the rows x own panel (column major).
struct Sn3 {
  int c0 = 0, n = 0;  // factor-order positions [c0, c0 + n)
  int parent = -1, ch[2] = {-1, -1}, nch = 0;
  int height = 0, depth = 0;
  int box[6] = {0, 0, 0, 0, 0, 0};  // x0, y0, z0, w, h, d of the nd call
  std::vector<int> rows;
};

struct Sym3 {
  int nn[3] = {0, 0, 0};
  int n = 0, nshell = 0;
  std::vector<int> perm, pinv;  // perm[pos] = window node
  std::vector<Sn3> sn;          // postorder
  int root = -1, max_height = 0, max_depth = 0;
  long nnz_ref = 0;             // nnz(L) + n, as the restatement counts it
  // per-class factor values: D at [0, n), then per supernode the packed
  // inverse diagonal block and the panel
  std::vector<long> linv_off, pan_off;
  long nvals = 0;
  long stored_lower = 0;        // strictly-lower entries stored (inverse blocks + panels)
  // forward update vectors (per RHS): r entries per supernode
  std::vector<long> upd_off;
  long nupd = 0;
  // front entry f (own columns, then rows) -> contributions of the children's
  // update vectors (absolute offsets into the per-RHS update array, -1: none)
  std::vector<long> cmap_off;   // per supernode, n + r entries
  std::vector<int> cmap0, cmap1;
  std::vector<long> rows_off;   // concatenated rows
  std::vector<int> rows_all;
  // numeric factorization: front of supernode s is (2n + r) x (n + r), column
  // major, rows = own, rows, and n identity rows E (L_E = L^-T D^-1 gives the
  // inverse of the diagonal block); its trailing r x r block is the
  // contribution block the parent extend-adds
  std::vector<long> front_off;
  long front_words = 0;
  std::vector<long> ext_off;    // per supernode (as a child): r parent front indices
  std::vector<int> ext;
  // assembled matrix entries per supernode: front (i, j), window node, kind
  // (0 diagonal, 1..6: -x +x -y +y -z +z neighbour of the column's node)
  std::vector<int> aent_ptr;
  std::vector<int> aent_i, aent_j, aent_node, aent_kind;
};

void build_sym3(int nx, int ny, int nz, Sym3& S);
std::vector<int> nd_order3(int nx, int ny, int nz);

struct Sub3 {
  int ix[3] = {0, 0, 0};
  int c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};
  int w0[3] = {0, 0, 0}, nn[3] = {0, 0, 0};
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  int own0[3] = {0, 0, 0}, own1[3] = {0, 0, 0};
  std::vector<double> w[3];  // blend weights per axis
  int cls = -1;
};

// stretch coefficients of one window (or the global box): per axis the nodal
// a and the inverse half-step 1/a, interleaved complex
struct Op3 {
  std::vector<double> an[3], iah[3];
};

struct Setup3 {
  double x0 = 0, y0 = 0, z0 = 0, h = 0;
  int m[3] = {0, 0, 0}, n[3] = {1, 1, 1}, nov = 0, nramp = 1;
  int ext = 0, gn[3] = {0, 0, 0}, mc[3] = {0, 0, 0};
  double omega = 0, velocity = 1, sigma0 = 0, k2 = 0;
  Op3 gop;
  std::vector<Sub3> subs;
  std::vector<Op3> subop;
  int ncls = 0;
  std::vector<int> cls_rep, cls_ptr, cls_members;
};

int build_setup3(const hddm3_problem& p, Setup3& S, std::string& msg);


}  // namespace hddm3
