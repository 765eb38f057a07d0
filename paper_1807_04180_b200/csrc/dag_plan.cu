// Host plan of the dataflow supernodal solve (dag.cuh): units, levels, partial
// slots, incoming-partial lists and the topologically ordered task list.
// Everything here is symbolic (one structure per window shape) except the tile
// list; it is built once per engine.
#include "dag_plan.h"

#include <algorithm>
#include <map>
#include <stdexcept>

namespace hddm {

namespace {

long long align16(long long v) { return (v + 15) & ~15LL; }
// staged units: positions' vectors + (forward) partials of the rows / (backward) x of the
// outside positions the rows reach
long long unit_core(const DagUnit& U, int M) {
  return align16((long long)(U.npos + std::max(U.nrow, U.nxe)) * M * (long long)sizeof(cplx));
}
long long unit_vals(const DagUnit& U) {
  return std::max(U.f1 - U.f0, U.b1 - U.b0) * (long long)sizeof(cplx);
}

}  // namespace

// two CTAs per SM: 2 x (dynamic + ~6 KB static + 1 KB reserved) <= 228 KB
int dag_smem_budget() { return 100 * 1024; }

// One decomposition: subtree units rooted at height hb, single units above.
static void build_dec(const Symbolic& Y, const std::vector<char>& live_sn, int hb, DagPlanHost::Dec& D) {
  const int nsn = int(Y.sn.size());
  D = DagPlanHost::Dec();
  D.hb = hb;
  std::vector<int> first(nsn);
  for (int s = 0; s < nsn; ++s) {  // postorder: children first
    first[s] = Y.sn[s].c0;
    for (int k = 0; k < Y.sn[s].nch; ++k) first[s] = std::min(first[s], first[Y.sn[s].child[k]]);
  }
  std::vector<int> unit_of(nsn, -1);
  std::vector<int> subtree_live(nsn, 0);
  for (int s = 0; s < nsn; ++s) subtree_live[s] = live_sn[s];  // live_sn is already subtree-wide
  for (int s = 0; s < nsn; ++s) {
    const SnNode& a = Y.sn[s];
    const bool single = a.height > hb;
    const bool sroot = !single && (a.parent < 0 || Y.sn[a.parent].height > hb);
    if (!single && !sroot) continue;
    DagUnit U{};
    U.kind = single ? 1 : 0;
    U.height = a.height;
    U.live = subtree_live[s];
    U.pos0 = single ? a.c0 : first[s];
    U.npos = a.c0 + a.n - U.pos0;
    // the unit's supernodes: single -> s; subtree -> every supernode whose c0 lies in
    // the position range (postorder: the subtree is contiguous, ending at s)
    std::vector<int> mem;
    if (single) {
      mem.push_back(s);
    } else {
      for (int d = 0; d <= s; ++d)
        if (Y.sn[d].c0 >= U.pos0 && Y.sn[d].c0 < U.pos0 + U.npos) mem.push_back(d);
    }
    const int uid = int(D.unit.size());
    for (int d : mem) unit_of[d] = uid;
    U.row0 = Y.sn[mem.front()].rs0;
    U.nrow = Y.sn[mem.back()].rs0 + Y.sn[mem.back()].nrs - U.row0;
    U.f0 = Y.sn[mem.front()].fdiag;
    U.f1 = Y.sn[mem.back()].fend;
    U.b0 = Y.sn[mem.front()].bdinv;
    U.b1 = Y.sn[mem.back()].bend;
    // levels by height, bottom-up
    std::map<int, std::vector<int>> byh;
    for (int d : mem) byh[Y.sn[d].height].push_back(d);
    U.lv0 = int(D.lv.size());
    for (auto& kv : byh) {
      DagLv L{};
      L.kind = Y.sn[kv.second.front()].kind;
      L.s0 = int(D.lsn.size());
      L.ns = int(kv.second.size());
      L.r0 = int(D.lrow.size());
      for (int d : kv.second) {
        if (Y.sn[d].kind != L.kind) throw std::runtime_error("dag plan: mixed leaf/separator level");
        D.lsn.push_back(d);
        D.lsr.push_back(L.nrow);
        for (int r = 0; r < Y.sn[d].nrs; ++r) {
          const int rr = Y.sn[d].rs0 + r;
          D.lrow.push_back(rr);
          D.lrm.push_back(Y.srow_dpos[rr]);
          D.lrm.push_back(Y.srow_first[rr]);
          D.lrm.push_back(int(Y.srow_boff[rr]));
          D.lrm.push_back(int(D.lsn.size()) - 1 - L.s0);  // the supernode's index in its level
        }
        L.nmax = std::max(L.nmax, Y.sn[d].n);
        L.rmax = std::max(L.rmax, Y.sn[d].nrs);
        L.nrow += Y.sn[d].nrs;
      }
      D.lv.push_back(L);
    }
    U.nlv = int(D.lv.size()) - U.lv0;
    D.unit.push_back(U);
  }
  for (int s = 0; s < nsn; ++s)
    if (unit_of[s] < 0) throw std::runtime_error("dag plan: supernode outside every unit");
  D.unit_of = unit_of;
  // partial slots: smem per row of a subtree unit; global per row of a single unit and
  // per distinct target outside a subtree unit (merged in row order)
  const int nrows = int(Y.srow_first.size());
  D.row_slot.assign(nrows, 0);
  int G = 0;
  std::vector<std::vector<std::pair<int, int>>> inc(Y.n);  // per position: (ref, source unit)
  for (size_t u = 0; u < D.unit.size(); ++u) {
    DagUnit& U = D.unit[u];
    if (U.kind == 1) {
      for (int r = U.row0; r < U.row0 + U.nrow; ++r) {
        const int g = G++;
        D.row_slot[r] = -(g + 1);
        inc[Y.srow_dpos[r]].push_back({-(g + 1), int(u)});
      }
      continue;
    }
    U.ex0 = int(D.ext.size());
    std::map<int, int> ext_of;  // target position -> ext index
    for (int r = U.row0; r < U.row0 + U.nrow; ++r) {
      const int slot = r - U.row0;
      D.row_slot[r] = slot;
      const int p = Y.srow_dpos[r];
      if (p >= U.pos0 && p < U.pos0 + U.npos) {
        inc[p].push_back({slot, -1});
        continue;
      }
      auto it = ext_of.find(p);
      if (it == ext_of.end()) {
        DagExt E{};
        E.gslot = G++;
        it = ext_of.emplace(p, int(D.ext.size())).first;
        D.ext.push_back(E);
        D.ext_tgt.push_back(p);
        inc[p].push_back({-(E.gslot + 1), int(u)});
      }
    }
    // sources of each merge in row order
    for (int e = U.ex0; e < int(D.ext.size()); ++e) {
      DagExt& E = D.ext[e];
      E.src0 = int(D.ext_src.size());
      for (int r = U.row0; r < U.row0 + U.nrow; ++r)
        if (Y.srow_dpos[r] == D.ext_tgt[e]) D.ext_src.push_back(r - U.row0);
      E.nsrc = int(D.ext_src.size()) - E.src0;
    }
    U.nex = int(D.ext.size()) - U.ex0;
  }
  D.G = G;
  D.in_ptr.assign(Y.n + 1, 0);
  for (int p = 0; p < Y.n; ++p) {
    D.in_ptr[p] = int(D.in_ref.size());
    for (auto& rs : inc[p]) {
      D.in_ref.push_back(rs.first);
      D.in_live.push_back(rs.second < 0 ? 1 : (unsigned char)D.unit[rs.second].live);
    }
  }
  D.in_ptr[Y.n] = int(D.in_ref.size());
  // per unit: the outside positions its rows reach (backward: their x is staged), and
  // per level row where its x comes from
  D.lrx.assign(D.lrow.size(), 0);
  for (DagUnit& U : D.unit) {
    U.xe0 = int(D.xe.size());
    std::map<int, int> idx;
    for (int l = U.lv0; l < U.lv0 + U.nlv; ++l) {
      const DagLv& L = D.lv[l];
      for (int f = L.r0; f < L.r0 + L.nrow; ++f) {
        const int p = Y.srow_dpos[D.lrow[f]];
        if (p >= U.pos0 && p < U.pos0 + U.npos) {
          D.lrx[f] = p - U.pos0;
          continue;
        }
        auto it = idx.find(p);
        if (it == idx.end()) {
          it = idx.emplace(p, int(D.xe.size()) - U.xe0).first;
          D.xe.push_back(p);
        }
        D.lrx[f] = -(it->second + 1);
      }
    }
    U.nxe = int(D.xe.size()) - U.xe0;
  }
}

// chunk lists of a streamed single unit (supernode s): the forward walks the panels
// of its diagonal block then the block rows column by column; the backward walks the
// block rows (each chunk with its rows' x) then the panels from the last
static void stream_chunks(const Symbolic& Y, int s, int M, long long bufe, std::vector<DagChunk>& ch,
                          std::vector<int>& meta, int& fc0, int& nfc, int& bc0, int& nbc) {
  const SnNode& a = Y.sn[s];
  const int n = a.n;
  const int nb = a.kind == 1 ? (n + kDiagBlk - 1) / kDiagBlk : 0;
  fc0 = int(ch.size());
  for (int b = 0; b < nb; ++b) {
    const int b0 = b * kDiagBlk, b1 = std::min(n, b0 + kDiagBlk), bw = b1 - b0;
    const long long po = a.fdiag + fpanel_off(n, b), xs = (long long)bw * (bw - 1) / 2;
    if (xs > 0) ch.push_back({po, int(xs), 0, b, b0, b1, -1});
    if (n > b1) {
      const int cpc = int(std::max<long long>(1, bufe / (n - b1)));
      for (int j = b0; j < b1; j += cpc) {
        const int je = std::min(b1, j + cpc);
        ch.push_back({po + xs + (long long)(j - b0) * (n - b1), (je - j) * (n - b1), 1, b, j, je, -1});
      }
    }
  }
  // block rows, column-major: column q holds the rows with first <= q; once per group
  // of kDagMG members (the accumulators live in registers)
  for (int g = 0; g * kDagMG < M; ++g) {
    int q = 0;
    while (q < n) {
      const long long o = Y.col_off[a.c0 + q];
      int qe = q;
      long long cnt = 0;
      while (qe < n) {
        const long long cq = (qe + 1 < n ? Y.col_off[a.c0 + qe + 1] : a.fend - a.frows) - Y.col_off[a.c0 + qe];
        if (qe > q && cnt + cq > bufe) break;
        cnt += cq;
        ++qe;
      }
      if (cnt > 0) ch.push_back({a.frows + o, int(cnt), 2, g, q, qe, -1});
      q = qe;
    }
  }
  nfc = int(ch.size()) - fc0;
  bc0 = int(ch.size());
  for (int g = 0; g * kDagMG < M; ++g) {  // block rows, row-major, with their x (M values
    int r = 0;                             // each) and (first, offset) pairs, per member group
    while (r < a.nrs) {
      int re = r;
      long long cnt = 0;
      while (re < a.nrs) {
        const long long len = n - Y.srow_first[a.rs0 + re];
        if (re > r && cnt + len + M + 1 > bufe) break;  // + 1: the pair (8 bytes) rounded up
        cnt += len + M + 1;
        ++re;
      }
      while (meta.size() % 4) meta.push_back(0);
      const int mo = int(meta.size());
      for (int q = r; q < re; ++q) {
        meta.push_back(Y.srow_first[a.rs0 + q]);
        meta.push_back(int(Y.srow_boff[a.rs0 + q] - Y.srow_boff[a.rs0 + r]));
      }
      ch.push_back({a.brows + Y.srow_boff[a.rs0 + r], int(cnt - (long long)(re - r) * (M + 1)), 3, g, r, re, mo});
      r = re;
    }
  }
  for (int b = nb - 1; b >= 0; --b) {
    const int b0 = b * kDiagBlk, b1 = std::min(n, b0 + kDiagBlk), bw = b1 - b0;
    const long long po = a.bdiag + bpanel_off(n, b), ls = (long long)bw * (n - b1);
    if (n > b1) {
      const int rpc = int(std::max<long long>(1, bufe / bw));
      for (int i = b1; i < n; i += rpc) {
        const int ie = std::min(n, i + rpc);
        ch.push_back({po + (long long)(i - b1) * bw, (ie - i) * bw, 4, b, i, ie, -1});
      }
    }
    const long long xs = (long long)bw * (bw - 1) / 2;
    if (xs > 0) ch.push_back({po + ls, int(xs), 5, b, b0, b1, -1});
  }
  nbc = int(ch.size()) - bc0;
}

long long DagPlanHost::Dec::finalize(int Mt, long long budget, const Symbolic& Y) {
  M = Mt;
  smem_need = 0;
  ch.clear();
  cmeta.clear();
  const long long huge = 1LL << 40;
  for (const DagLv& L : lv)
    if ((L.kind == 1 && (long long)L.ns * std::min(L.nmax, kDiagBlk) * M > 4LL * kDagThreads) ||
        L.ns > 64)  // blocked diagonal: <= 4 results per thread; kLvSn supernodes per level
      return smem_need = huge;
  for (DagUnit& U : unit) {
    const long long core = unit_core(U, M), vals = unit_vals(U);
    const long long cofb = align16((long long)U.npos * sizeof(int));
    U.fc0 = U.nfc = U.bc0 = U.nbc = 0;
    if (core + vals + cofb <= budget) {
      U.voff = int(core);
      U.cof = int(core + vals);
      U.cap = U.nrow;
      smem_need = std::max(smem_need, core + vals + cofb);
      if (U.nxe > 4096) return smem_need = huge;  // bulk loads issued by one warp
    } else if (U.kind == 0) {
      return smem_need = huge;  // subtree units run from shared memory
    } else {
      // streamed: the supernode's vectors, its column offsets, two chunk buffers
      U.voff = -1;
      const int s = lsn[lv[U.lv0].s0];
      const long long vec = align16((long long)U.npos * M * (long long)sizeof(cplx));
      U.cof = int(vec);
      U.buf = int(vec + cofb);
      const long long bufb = ((budget - U.buf) / 2) & ~15LL;
      U.bufb = int(bufb);
      const long long bufe = bufb / (long long)sizeof(cplx);
      const long long mg = std::min(M, kDagMG);
      if (bufe < 4LL * std::max(kDiagBlk, M) || U.npos * mg > (long long)kDagAcc * kDagThreads ||
          (long long)U.nrow * mg > (long long)kDagAcc * kDagThreads || U.nrow > bufe)
        return smem_need = huge;  // register accumulators: <= kDagAcc items per thread
      if (Y.sn[s].kind != 1) return smem_need = huge;
      // the forward gathers its incoming partial refs into a chunk buffer first
      if (in_ptr[Y.sn[s].c0 + Y.sn[s].n] - in_ptr[Y.sn[s].c0] > bufe * 4) return smem_need = huge;
      stream_chunks(Y, s, M, bufe, ch, cmeta, U.fc0, U.nfc, U.bc0, U.nbc);
      for (int q = 0; q < 4; ++q) cmeta.push_back(0);  // bulk copies round up to 16 bytes
      smem_need = std::max(smem_need, (long long)U.buf + 2 * bufb);
    }
  }
  return smem_need;
}

void build_dag_plan(const Symbolic& Y, const std::vector<char>& live_sn,
                    const std::vector<DagTileIn>& tiles, DagPlanHost& P) {
  P = DagPlanHost();
  const int nsn = int(Y.sn.size());
  P.sn.resize(nsn);
  for (int s = 0; s < nsn; ++s) {
    const SnNode& a = Y.sn[s];
    DagSn& d = P.sn[s];
    d.kind = a.kind;
    d.c0 = a.c0;
    d.n = a.n;
    d.lw = a.kind == 0 ? a.w : 0;
    d.rs0 = a.rs0;
    d.nrs = a.nrs;
    d.fdiag = a.fdiag;
    d.frows = a.frows;
    d.bdinv = a.bdinv;
    d.bdiag = a.bdiag;
    d.brows = a.brows;
  }
  P.row_first = Y.srow_first;
  P.row_dpos = Y.srow_dpos;
  P.row_boff.assign(Y.srow_boff.begin(), Y.srow_boff.end());
  P.col_off = Y.col_off;
  const long long budget = dag_smem_budget();
  // one decomposition per distinct tile width: the highest hb whose subtree units
  // (vectors, partials and factor values) fit the shared-memory budget
  std::map<int, int> dec_of_M;
  for (const DagTileIn& t : tiles) {
    if (t.M < 1 || t.M > kDagMaxM) throw std::runtime_error("dag plan: tile width out of range");
    if (dec_of_M.count(t.M)) continue;
    int best = -1;
    DagPlanHost::Dec D;
    for (int hb = 0; hb <= Y.max_height; ++hb) {
      build_dec(Y, live_sn, hb, D);
      if (D.finalize(t.M, budget, Y) <= budget) best = hb;
      else break;
    }
    if (best < 0) throw std::runtime_error("dag plan: no unit decomposition fits shared memory");
    if (P.dec.size() == size_t(kDagDecs)) throw std::runtime_error("dag plan: too many tile widths");
    build_dec(Y, live_sn, best, D);
    D.finalize(t.M, budget, Y);
    dec_of_M[t.M] = int(P.dec.size());
    P.dec.push_back(D);
  }
  for (auto& D : P.dec) {
    D.lvsn.clear();
    for (int d : D.lsn) D.lvsn.push_back(P.sn[d]);
  }
  // tiles: widest first (their chains are the longest)
  std::vector<int> order(tiles.size());
  for (size_t k = 0; k < tiles.size(); ++k) order[k] = int(k);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tiles[a].M > tiles[b].M; });
  long long pb = 0;
  for (int k : order) {
    const DagTileIn& t = tiles[k];
    DagTile T{};
    T.cb = t.cb;
    T.c = t.c;
    T.m = t.m;
    T.M = t.M;
    T.dec = dec_of_M[t.M];
    T.pbase = pb;
    pb += (long long)P.dec[T.dec].G * t.M;
    for (int i = 0; i < kDagMaxM; ++i) T.t[i] = t.t[std::min(i, t.M - 1)];
    P.tile.push_back(T);
  }
  P.nP = pb;
  P.smem_bytes = 0;
  for (const auto& D : P.dec) P.smem_bytes = std::max(P.smem_bytes, D.smem_need);
  // tasks: forward by unit height ascending, then backward by height descending;
  // within a height, tiles in the order above
  struct Key {
    int kind, h, tile, unit;
  };
  std::vector<Key> keys;
  for (size_t ti = 0; ti < P.tile.size(); ++ti) {
    const auto& D = P.dec[P.tile[ti].dec];
    for (size_t u = 0; u < D.unit.size(); ++u) {
      keys.push_back({0, D.unit[u].height, int(ti), int(u)});
      keys.push_back({1, D.unit[u].height, int(ti), int(u)});
    }
  }
  std::stable_sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
    if (a.kind != b.kind) return a.kind < b.kind;
    if (a.h != b.h) return a.kind == 0 ? a.h < b.h : a.h > b.h;
    return a.tile < b.tile;
  });
  std::map<long long, int> idx;  // (kind, tile, unit) -> task
  auto key_of = [](int kind, int tile, int unit) {
    return ((long long)kind << 50) | ((long long)tile << 25) | (long long)unit;
  };
  for (size_t k = 0; k < keys.size(); ++k) idx[key_of(keys[k].kind, keys[k].tile, keys[k].unit)] = int(k);
  P.task.resize(keys.size());
  for (size_t k = 0; k < keys.size(); ++k) {
    const Key& K = keys[k];
    const auto& D = P.dec[P.tile[K.tile].dec];
    const DagUnit& U = D.unit[K.unit];
    DagTask T{};
    T.kind = K.kind;
    T.tile = K.tile;
    T.unit = K.unit;
    T.dep0 = T.dep1 = -1;
    // the unit's root supernode: the last one (postorder)
    const int root = D.lsn[D.lv[U.lv0 + U.nlv - 1].s0 + D.lv[U.lv0 + U.nlv - 1].ns - 1];
    const SnNode& r = Y.sn[root];
    if (K.kind == 0) {
      if (U.kind == 1) {
        int nd = 0;
        for (int c = 0; c < r.nch; ++c) {
          const int cu = D.unit_of[r.child[c]];
          const int dep = idx.at(key_of(0, K.tile, cu));
          (nd++ == 0 ? T.dep0 : T.dep1) = dep;
        }
      }
    } else {
      T.dep0 = r.parent >= 0 ? idx.at(key_of(1, K.tile, D.unit_of[r.parent]))
                             : idx.at(key_of(0, K.tile, K.unit));
    }
    if ((T.dep0 >= int(k)) || (T.dep1 >= int(k))) throw std::runtime_error("dag plan: task order");
    P.task[k] = T;
  }
}

}  // namespace hddm
