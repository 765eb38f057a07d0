// Dataflow (task-DAG) supernodal solve: tables shared by the host plan builder
// (dag_plan.cpp) and the persistent kernel (kernels_dag.cu).
//
// The ND tree of the window (one symbolic structure for every class) is cut into
// UNITS: the subtrees rooted at height hb (processed whole inside one CTA, their
// internal partial sums in shared memory) and every supernode above hb (a unit of
// its own). A task is (tile, unit, sweep); a persistent grid takes tasks from an
// atomic ticket in topological order and waits only for the task's own
// predecessors (children's forward, parent's backward) -- no level-wide barriers
// and no kernel boundaries inside the solve. hb is chosen per tile width M so a
// unit's vectors and partial sums fit the shared-memory budget.
#pragma once

#include "dev.cuh"

namespace hddm {

constexpr int kDagThreads = 256;
constexpr int kDagMaxM = 16;  // members per tile (registers: M accumulators per thread)
constexpr int kDagDecs = 4;   // unit decompositions (distinct hb) per plan
constexpr int kDagMG = 8;     // streamed units: members per register group
constexpr int kDagAcc = 8;    // streamed units: accumulator items per thread

struct DagSn {  // per supernode (symbolic; value offsets are per class)
  int kind, c0, n, lw;  // kind 0 leaf (band, natural order, width lw), 1 separator
  int rs0, nrs;         // block rows, sorted by first column (row tables below)
  int pad0, pad1;
  long long fdiag, frows;         // forward copy F: diag (col-major / band), rows col-major
  long long bdinv, bdiag, brows;  // backward copy B: 1/D, diag (row-major / band), rows row-major
  long long pad2;
};

struct DagLv {  // one level (height) of a unit
  int kind;     // 0 leaves, 1 separators
  int s0, ns;   // supernodes: lsn[s0 .. s0 + ns)
  int nmax;     // largest n of them
  int rmax;     // most block rows of them
  int nrow;     // block rows of all of them
  int r0;       // their rows: lrow[r0 .. r0 + nrow), supernode si's from lsr[s0 + si]
  int pad;
};

struct DagUnit {
  int kind;           // 0 subtree (shared-memory partials), 1 single supernode
  int pos0, npos;     // its positions (contiguous in factor order)
  int lv0, nlv;       // levels, bottom-up
  int row0, nrow;     // its supernodes' sorted rows (contiguous); smem slot = row - row0
  int ex0, nex;       // merges of partials leaving the unit (subtree units)
  int live;           // steps >= 2: the subtree holds transfer-patch nodes
  int height;
  int voff;           // >= 0: the sweep's factor values are staged (one bulk copy) at this
                      // byte offset of shared memory; -1: streamed from global memory
  int cap;            // backward: rows staged per chunk
  int cof;            // staged units: byte offset of the positions' column offsets (forward)
  int xe0, nxe;       // staged units: positions outside the unit its rows reach (xe list);
                      // their x is bulk-loaded with the unit's z at the backward's start
  int fc0, nfc;       // streamed units: forward chunks ch[fc0 .. fc0 + nfc)
  int bc0, nbc;       // streamed units: backward chunks
  int buf;            // streamed units: byte offset of the two chunk buffers (each bufb)
  int bufb;
  long long f0, f1;   // forward-copy value range (per class), for the L2 prefetch
  long long b0, b1;   // backward-copy value range
};

// A chunk of a streamed unit's factor values, bulk-copied into one of two shared-
// memory buffers. Forward kinds: 0 Xinv of panel b, 1 columns [a, z) of the rows
// below panel b, 2 columns [a, z) of the block rows (push); backward kinds: 3 block
// rows [a, z) (with their x), 4 rows [a, z) below panel b, 5 Xinv of panel b.
// Kinds 2 and 3 carry the member group in b (members [kDagMG b, kDagMG (b + 1))).
struct DagChunk {
  long long off;  // per-class offset in the sweep's copy
  int cnt;        // complex values
  int kind, b, a, z;
  int meta;       // kind 3: offset (ints, 16-byte aligned) of its rows' (first, offset) pairs
};

struct DagExt {  // a global slot = sum of smem slots ext_src[src0 .. src0 + nsrc) in order
  int gslot, src0, nsrc, pad;
};

struct DagTask {
  int kind;   // 0 forward, 1 backward
  int tile, unit;
  int dep0, dep1;  // task indices this one waits for (-1: none)
  int pad;
};

struct DagDec {  // one unit decomposition
  const DagUnit* unit;
  const DagLv* lv;
  const DagSn* lvsn;    // supernodes per level (copies)
  const int* lsr;       // per level supernode: offset of its rows in the level's row list
  const int4* lrm;      // per level row (concatenated per supernode): (dpos, first, boff, si)
  const int* lrx;       // per level row: >= 0 position inside the unit (dpos - pos0),
                        // < 0: -(e + 1), e its index in the unit's xe list
  const int* xe;        // per unit: the outside positions its rows reach
  const DagChunk* ch;   // streamed units' chunk lists
  const int* cmeta;     // kind-3 chunk metadata
  const int* row_slot;  // per sorted row: >= 0 smem slot, < 0 global slot -(g + 1)
  const int* in_ptr;    // per position: incoming partial refs in_ref[in_ptr[p] .. in_ptr[p + 1])
  const int* in_ref;    // >= 0 smem slot, < 0 global slot -(g + 1)
  const unsigned char* in_live;  // per ref: its source unit is live (steps >= 2)
  const DagExt* ext;
  const int* ext_src;
  int G;                // global slots
  int hb;
};

struct DagTile {  // up to kDagMaxM members of one class
  long long cb;     // storage offset of (position 0, first member of the tile)
  long long pbase;  // partial-slot base (complex): slot g, member k at pbase + g * M + k
  int c, m, M, dec;  // class, class member count (vector stride), tile members, decomposition
  int t[kDagMaxM];   // subdomain of each member
};

struct DagArgs {
  const DagSn* sn;
  const int* row_first;        // per sorted row
  const int* row_dpos;
  const long long* row_boff;   // offset of entry [first] relative to brows
  const int* col_off;          // per position: its column's offset relative to frows
  DagDec dec[kDagDecs];
  const DagTile* tile;
  const DagTask* task;
  int ntask;
  int* ticket;  // zeroed before each launch
  int* done;    // ntask flags, zeroed before each launch
  const cplx* vF;
  const cplx* vB;
  long long nvF, nvB;
  const int* flag;  // RHS t active iff (flag[t] != 0) == flag_on
  int flag_on;
  int sparse;       // right-hand sides nonzero only on the transfer patches (steps >= 2)
  const cplx* B;
  cplx* X;
  cplx* P;          // partial slots
  int smem_bytes;
  long long* prof;  // profiling builds: 8 categories x 8 counters (cycles per phase, tasks)
  long long* trace; // profiling builds: per task (start ns, end ns, SM, CTA)
};

}  // namespace hddm
