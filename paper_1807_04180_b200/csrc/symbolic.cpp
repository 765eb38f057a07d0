// Host symbolic analysis: the reference's elimination order, the nested-
// dissection supernode tree, the exact nonzero profile of L and the GPU value
// layout. Computed once per window shape (all windows of a partition share it,
// proj/src/partition.cpp:68).
//
// Elimination order: ring first (bottom row, side columns row by row, top row),
// then recursive bisection with the separator after both halves and leaves of
// at most 6x6 in natural order -- exactly grid_nd_order/nd_rec
// (proj/src/sparse.cpp:20-57). Pivots are never reordered: supernodes are the
// nd_rec calls themselves, so the numeric factor is the reference's LDL^T
// (sparse.cpp:110-174) up to rounding.
#include <algorithm>
#include <cstdio>
#include <stdexcept>

#include "hddm_internal.h"

namespace hddm {

namespace {

struct TreeBuilder {
  int nx;
  std::vector<int>& order;
  std::vector<SnNode>& sn;

  // returns supernode index or -1 (empty region)
  int rec(int x0, int y0, int w, int h) {
    if (w <= 0 || h <= 0) return -1;
    SnNode node;
    node.x0 = x0;
    node.y0 = y0;
    node.w = w;
    node.h = h;
    if (w <= 6 && h <= 6) {
      node.kind = 0;
      node.c0 = int(order.size());
      for (int q = y0; q < y0 + h; ++q)
        for (int p = x0; p < x0 + w; ++p) order.push_back(q * nx + p);
    } else {
      int a, b;
      std::vector<int> sep;
      if (w >= h) {
        const int mid = x0 + w / 2;
        a = rec(x0, y0, mid - x0, h);
        b = rec(mid + 1, y0, x0 + w - mid - 1, h);
        for (int q = y0; q < y0 + h; ++q) sep.push_back(q * nx + mid);
      } else {
        const int mid = y0 + h / 2;
        a = rec(x0, y0, w, mid - y0);
        b = rec(x0, mid + 1, w, y0 + h - mid - 1);
        for (int p = x0; p < x0 + w; ++p) sep.push_back(mid * nx + p);
      }
      node.kind = 1;
      node.c0 = int(order.size());
      order.insert(order.end(), sep.begin(), sep.end());
      for (int c : {a, b})
        if (c >= 0) node.child[node.nch++] = c;
    }
    node.n = int(order.size()) - node.c0;
    sn.push_back(node);
    const int id = int(sn.size()) - 1;
    for (int k = 0; k < sn[id].nch; ++k) sn[sn[id].child[k]].parent = id;
    return id;
  }
};

void ring_order(int nx, int ny, std::vector<int>& order) {
  for (int p = 0; p < nx; ++p) order.push_back(p);
  for (int q = 1; q < ny - 1; ++q) {
    order.push_back(q * nx);
    order.push_back(q * nx + nx - 1);
  }
  for (int p = 0; p < nx; ++p) order.push_back((ny - 1) * nx + p);
}

}  // namespace

std::vector<int> nd_order(int nx, int ny) {
  std::vector<int> order;
  order.reserve(size_t(nx) * ny);
  if (nx <= 2 || ny <= 2) {
    for (int k = 0; k < nx * ny; ++k) order.push_back(k);
    return order;
  }
  ring_order(nx, ny, order);
  std::vector<SnNode> sn;
  TreeBuilder tb{nx, order, sn};
  tb.rec(1, 1, nx - 2, ny - 2);
  return order;
}

void build_symbolic(int nx, int ny, Symbolic& S) {
  if (nx <= 2 || ny <= 2) throw std::runtime_error("window too small for the ND solver");
  S = Symbolic();
  S.nx = nx;
  S.ny = ny;
  S.n = nx * ny;
  const int n = S.n;
  S.perm.reserve(n);
  ring_order(nx, ny, S.perm);
  S.nring = int(S.perm.size());
  TreeBuilder tb{nx, S.perm, S.sn};
  const int root = tb.rec(1, 1, nx - 2, ny - 2);
  if (int(S.perm.size()) != n) throw std::runtime_error("ND order is not a permutation");
  S.pinv.assign(n, -1);
  for (int k = 0; k < n; ++k) S.pinv[S.perm[k]] = k;
  const int nsn = int(S.sn.size());
  S.sn_of_pos.assign(n, -1);
  for (int s = 0; s < nsn; ++s)
    for (int k = 0; k < S.sn[s].n; ++k) S.sn_of_pos[S.sn[s].c0 + k] = s;
  // heights (postorder) and depths (reverse postorder)
  for (int s = 0; s < nsn; ++s) {
    int hgt = 0;
    for (int k = 0; k < S.sn[s].nch; ++k) hgt = std::max(hgt, S.sn[S.sn[s].child[k]].height + 1);
    S.sn[s].height = hgt;
    S.max_height = std::max(S.max_height, hgt);
  }
  S.sn[root].depth = 0;
  for (int s = nsn - 1; s >= 0; --s)
    if (S.sn[s].parent >= 0) {
      S.sn[s].depth = S.sn[S.sn[s].parent].depth + 1;
      S.max_depth = std::max(S.max_depth, S.sn[s].depth);
    }

  // adjacency of A in factor order: interior 5-point couplings (ring rows are
  // identity and interior rows drop ring columns, discretize.cpp:98-160)
  auto interior = [&](int p, int q) { return p > 0 && q > 0 && p < nx - 1 && q < ny - 1; };
  std::vector<int> adj(size_t(4) * n, -1);
  for (int q = 1; q < ny - 1; ++q)
    for (int p = 1; p < nx - 1; ++p) {
      const int v = S.pinv[q * nx + p];
      const int nb[4][2] = {{p - 1, q}, {p + 1, q}, {p, q - 1}, {p, q + 1}};
      for (int d = 0; d < 4; ++d)
        if (interior(nb[d][0], nb[d][1])) adj[size_t(4) * v + d] = S.pinv[nb[d][1] * nx + nb[d][0]];
    }
  // elimination tree (Liu, with path compression)
  std::vector<int> parent(n, -1), anc(n, -1);
  for (int k = 0; k < n; ++k)
    for (int d = 0; d < 4; ++d) {
      int i = adj[size_t(4) * k + d];
      while (i >= 0 && i < k) {
        const int nxt = anc[i];
        anc[i] = k;
        if (nxt == -1) parent[i] = k;
        i = nxt;
      }
    }
  // row patterns -> per-(supernode, row) first column and count; leaf bands
  struct RowRec {
    int r, first, cnt;
  };
  std::vector<std::vector<RowRec>> srow(nsn);
  std::vector<int> mark(n, -1), touched;
  std::vector<int> sfirst(nsn, 0), scnt(nsn, 0), slast(nsn, -1);
  std::vector<int> band_first(n, -1), band_cnt(n, 0);
  long nnzL = 0;
  std::vector<int> stack;
  for (int k = S.nring; k < n; ++k) {
    mark[k] = k;
    touched.clear();
    const int sk = S.sn_of_pos[k];
    for (int d = 0; d < 4; ++d) {
      int i = adj[size_t(4) * k + d];
      if (i < 0 || i > k) continue;
      for (; i >= 0 && mark[i] != k; i = parent[i]) {
        mark[i] = k;
        ++nnzL;
        const int s = S.sn_of_pos[i];
        if (s == sk) {  // inside the diagonal block of the row's own supernode
          if (band_first[k] < 0 || i < band_first[k]) band_first[k] = i;
          ++band_cnt[k];
          continue;
        }
        if (slast[s] != k) {
          slast[s] = k;
          sfirst[s] = i;
          scnt[s] = 0;
          touched.push_back(s);
        }
        sfirst[s] = std::min(sfirst[s], i);
        ++scnt[s];
      }
    }
    for (int s : touched) srow[s].push_back({k, sfirst[s], scnt[s]});
  }
  S.nnz_ref = nnzL + n;

  // blocks: group each supernode's off-diagonal rows by owning ancestor
  S.blk.clear();
  S.row_first.clear();
  S.row_off.clear();
  S.nnz_stored = 0;
  for (int s = 0; s < nsn; ++s) {
    SnNode& nd = S.sn[s];
    if (nd.kind == 0) {
      nd.drow0 = int(S.row_first.size());
      for (int i = 0; i < nd.n; ++i) {
        const int k = nd.c0 + i;
        const int f = band_first[k] < 0 ? nd.n : band_first[k] - nd.c0;
        // contiguous profile assumed; padding keeps correctness otherwise
        S.row_first.push_back(std::min(f, i));
        S.row_off.push_back(0);
      }
    }
    nd.blk0 = int(S.blk.size());
    nd.rows.clear();
    const auto& rr = srow[s];
    size_t a = 0;
    while (a < rr.size()) {
      const int owner = S.sn_of_pos[rr[a].r];
      size_t b = a;
      while (b + 1 < rr.size() && S.sn_of_pos[rr[b + 1].r] == owner) ++b;
      Block B;
      B.src = s;
      B.dst = owner;
      const int rmin = rr[a].r, rmax = rr[b].r;
      B.r0 = rmin - S.sn[owner].c0;
      B.nr = rmax - rmin + 1;
      B.row0 = int(S.row_first.size());
      B.front0 = nd.n + int(nd.rows.size());
      size_t c = a;
      for (int r = rmin; r <= rmax; ++r) {
        int first = nd.n;  // padding row: empty
        if (c <= b && rr[c].r == r) {
          first = rr[c].first - nd.c0;
          ++c;
        }
        S.row_first.push_back(first);
        S.row_off.push_back(0);
        nd.rows.push_back(r);
      }
      S.blk.push_back(B);
      a = b + 1;
    }
    nd.nblk = int(S.blk.size()) - nd.blk0;
  }
  // incoming rows per destination position, in source (postorder) order
  std::vector<std::vector<int>> incoming(n);
  for (const Block& B : S.blk)
    for (int r = 0; r < B.nr; ++r) incoming[S.sn[B.dst].c0 + B.r0 + r].push_back(B.row0 + r);
  // value layout per supernode: [1/D | diagonal part | incoming runs of its rows]
  // -- every separator row's incoming entries form ONE contiguous run, so the
  // forward pull streams it; the backward reads each block row (a piece of some
  // ancestor's run) through the row table.
  long off = 0;
  S.run_off.assign(n + 1, 0);
  S.seg_ptr.assign(n + 1, 0);
  S.seg.clear();
  for (int s = 0; s < nsn; ++s) {
    SnNode& nd = S.sn[s];
    nd.dinv_off = off;
    off += nd.n;
    nd.diag_off = off;
    if (nd.kind == 1) {
      off += long(nd.n) * (nd.n - 1) / 2;
      S.nnz_stored += long(nd.n) * (nd.n - 1) / 2;
    } else {
      for (int i = 0; i < nd.n; ++i) {
        const int rt = nd.drow0 + i;
        S.row_off[rt] = off;
        off += i - S.row_first[rt];
        S.nnz_stored += i - S.row_first[rt];
      }
    }
  }
  std::vector<int> src_of(S.row_first.size(), -1);
  for (size_t b = 0; b < S.blk.size(); ++b)
    for (int r = 0; r < S.blk[b].nr; ++r) src_of[S.blk[b].row0 + r] = S.blk[b].src;
  for (int pos = 0; pos < n; ++pos) {
    S.run_off[pos] = off;
    S.seg_ptr[pos] = int(S.seg.size());
    for (int rt : incoming[pos]) {
      const SnNode& src = S.sn[src_of[rt]];
      const int len = src.n - S.row_first[rt];
      S.row_off[rt] = off;
      if (len > 0) S.seg.push_back({len, src.c0 + S.row_first[rt]});
      off += len;
      S.nnz_stored += len;
    }
  }
  S.run_off[n] = off;
  S.seg_ptr[n] = int(S.seg.size());
  S.nvals = off;

  // fronts, extend-add maps, A scatter lists
  S.front_words = 0;
  S.extadd.clear();
  S.aent0.assign(nsn + 1, 0);
  S.aent_i.clear();
  S.aent_j.clear();
  S.aent_node.clear();
  S.aent_kind.clear();
  for (int s = 0; s < nsn; ++s) {
    SnNode& nd = S.sn[s];
    const long F = nd.n + long(nd.rows.size());
    nd.front_off = S.front_words;
    S.front_words += F * F;
    auto loc = [&](int r) -> int {
      if (r >= nd.c0 && r < nd.c0 + nd.n) return r - nd.c0;
      auto it = std::lower_bound(nd.rows.begin(), nd.rows.end(), r);
      if (it == nd.rows.end() || *it != r) return -1;
      return nd.n + int(it - nd.rows.begin());
    };
    for (int k = 0; k < nd.nch; ++k) {
      SnNode& ch = S.sn[nd.child[k]];
      ch.extadd0 = int(S.extadd.size());
      ch.nextadd = int(ch.rows.size());
      for (int r : ch.rows) {
        const int l = loc(r);
        if (l < 0) throw std::runtime_error("child update row outside parent front");
        S.extadd.push_back(l);
      }
    }
    S.aent0[s] = int(S.aent_i.size());
    for (int k = 0; k < nd.n; ++k) {
      const int v = nd.c0 + k;
      S.aent_i.push_back(k);
      S.aent_j.push_back(k);
      S.aent_node.push_back(S.perm[v]);
      S.aent_kind.push_back(0);
      for (int d = 0; d < 4; ++d) {
        const int u = adj[size_t(4) * v + d];
        if (u < 0 || u < v) continue;
        const int l = loc(u);
        if (l < 0) throw std::runtime_error("matrix entry outside front");
        S.aent_i.push_back(l);
        S.aent_j.push_back(k);
        S.aent_node.push_back(S.perm[v]);
        S.aent_kind.push_back(1 + d);
      }
    }
  }
  S.aent0[nsn] = int(S.aent_i.size());

}

}  // namespace hddm
