// Internal host-side structures of the B200 DDM engine (not part of the C-ABI).
//
// Layout summary (DESIGN.md has the full story):
//  * every subdomain window has the same node counts (partition.cpp:68), so ONE
//    symbolic structure (reference elimination order, supernode tree, L profile)
//    serves every class;
//  * per-subdomain vectors live in the reference's elimination order
//    ("factor order", sparse.cpp:42-57) so supernodes are contiguous ranges;
//  * global fields are row-major, x fastest (types.hpp:37-56).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "hddm.h"

namespace hddm {

// Profiling knobs that change what the engine computes (leaving kernel families or
// stages out, timing aids): read only in builds compiled with -DHDDM_PROFILING
// (make EXTRA=-DHDDM_PROFILING); in the product library they are ignored, so a stray
// environment variable cannot change results. Tuning knobs that select between
// equivalent algorithms (tile sizes, lane shapes) are read in every build.
inline const char* profiling_env(const char* name) {
#ifdef HDDM_PROFILING
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// ------------------------------------------------------------------ symbolic
// One node of the nested-dissection tree produced by the reference's nd_rec
// (proj/src/sparse.cpp:20-40): a leaf block (natural order inside) or a
// separator line eliminated after both halves.
struct SnNode {
  int kind = 0;              // 0 leaf (band diag solve), 1 separator (dense inverse)
  int x0 = 0, y0 = 0, w = 0, h = 0;  // region of the nd_rec call (window-local nodes)
  int c0 = 0, n = 0;         // factor-order positions [c0, c0+n)
  int parent = -1;
  int child[2] = {-1, -1};
  int nch = 0;
  int height = 0;            // 0 for leaves; 1 + max child height
  int depth = 0;             // 0 at the root
  // front = [own columns] ++ rows[]  (rows: factor-order positions, ascending)
  std::vector<int> rows;
  int blk0 = 0, nblk = 0;    // outgoing blocks (L rows owned by ancestors)
  long diag_off = 0;         // sep: packed strictly-lower inverse; leaf: band entries
  long dinv_off = 0;         // 1/D, n entries
  int drow0 = 0;             // leaf: first row-table entry of its band rows
  long front_off = 0;        // workspace offset of the (n+rows) x (n+rows) front
  int nextadd = 0, extadd0 = 0;  // index maps for the children's update blocks
};

// Rows [r0, r0+nr) (relative to dst.c0) of ancestor `dst` against the columns of
// `src`. Row r stores columns [first[r], src.n) contiguously (profile storage).
struct Block {
  int src = 0, dst = 0, r0 = 0, nr = 0;
  int row0 = 0;    // first entry in the row tables
  int front0 = 0;  // front-row index (in src's front) of block row 0
};

struct Symbolic {
  int nx = 0, ny = 0, n = 0, nring = 0;
  std::vector<int> perm, pinv;       // perm[pos] = window node, pinv[node] = pos
  std::vector<SnNode> sn;            // postorder (children before parents)
  std::vector<int> sn_of_pos;        // supernode owning each interior position
  std::vector<Block> blk;
  std::vector<int> row_first;        // per block/band row: first column (relative)
  std::vector<long> row_off;         // per block/band row: value offset
  // forward runs: incoming entries of factor-order position p are the values
  // [run_off[p], run_off[p+1]), split into segments seg[seg_ptr[p]..seg_ptr[p+1])
  // of (length, first source position)
  struct Seg {
    int len, zbase;
  };
  std::vector<long> run_off;
  std::vector<int> seg_ptr;
  std::vector<Seg> seg;
  long nvals = 0;                    // complex values per class
  long nnz_ref = 0;                  // reference's factor_nonzeros() (nnz(L) + n)
  long nnz_stored = 0;               // strictly-lower entries actually stored
  int max_height = 0, max_depth = 0;
  long front_words = 0;              // complex words of front workspace per class
  std::vector<int> extadd;           // child front row -> parent front index
  // A scatter list: per supernode, entries (front i, front j) with i >= j
  std::vector<int> aent0;            // size sn+1
  std::vector<int> aent_i, aent_j;   // front indices
  std::vector<int> aent_node, aent_kind;  // window node, 0 diag 1 W 2 E 3 S 4 N
};

void build_symbolic(int nx, int ny, Symbolic& S);
std::vector<int> nd_order(int nx, int ny);

// ------------------------------------------------------------------ problem
struct Medium {
  int kind = 0;  // 0 constant, 1 layered, 2 lens
  double omega = 0, velocity = 1;
  std::vector<double> ylo, yhi, c;
  double bx0 = 0, bx1 = 0, by0 = 0, by1 = 0, margin = 0;
  double lamp = 0, lxc = 0, lyc = 0, lw = 1;
  double cmin = 1, cmax = 1;
};

struct Sub {
  int i = 0, j = 0, cx0 = 0, cx1 = 0, cy0 = 0, cy1 = 0;
  int wx0 = 0, wy0 = 0, nx = 0, ny = 0;
  bool lint = false, rint = false, bint = false, tint = false;
  std::vector<double> wx, wy;
  int own[4] = {0, 0, 0, 0};
  int cls = -1;
};

// Operator coefficient arrays of one window (DiscreteOperator,
// proj/include/helmddm/discretize.hpp:32-40): interleaved complex.
struct WinOp {
  std::vector<double> a1n, ia1h, a2n, ia2h;  // 2*nx, 2*nx, 2*ny, 2*ny (last half unused)
};

struct Setup {
  double x0 = 0, y0 = 0, h = 0;
  int mx = 0, my = 0, n1 = 1, n2 = 1, nov = 0, nramp = 1;
  int ext = 0, gnx = 0, gny = 0, mcx = 0, mcy = 0;
  double sigma0 = 0, c_sigma = 25;
  Medium med;
  WinOp gop;                      // global operator 1-D arrays
  std::vector<double> k2;         // global nodal k^2 (gnx*gny)
  std::vector<Sub> subs;
  std::vector<WinOp> subop;       // per subdomain
  int ncls = 0;
  std::vector<int> cls_rep;       // representative subdomain per class
  std::vector<int> cls_members;   // CSR over classes
  std::vector<int> cls_ptr;
};

// returns 0 or an error code (2 config, 1 other) with msg filled
int build_setup(const hddm_problem& p, Setup& S, std::string& msg);

}  // namespace hddm
