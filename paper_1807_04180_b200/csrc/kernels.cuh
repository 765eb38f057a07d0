// Kernel argument blocks and launcher prototypes (host <-> .cu glue).
#pragma once

#include <map>
#include <utility>
#include <vector>

#include "dev.cuh"

namespace hddm {

// fixed grid of the reduction kernels (4 x 148 SMs) => fixed summation order
constexpr int kReduceBlocks = 592;

// ------------------------------------------------------------------ solves
struct SolveArgs {
  const DevSn* sn;
  const DevBlk* blk;
  const int* row_first;
  const long long* row_off;
  const long long* run_off;  // per position: incoming run [run_off[p], run_off[p+1])
  const int* seg_ptr;        // per position: segments of the run
  const int2* seg;           // (length, first source position)
  const int* bw_ptr;         // per supernode: backward rows
  const BwRow* bw;
  const int* bw_cnt;         // per factor position (column): its supernode's backward rows that
                             // reach it (rows with first <= column; the lists are sorted by first)
  const SegRec* fseg;  // forward run segments of the plan in use (full or sparse RHS)
  const cplx* vals;    // ncls x nvals
  long long nvals;
  const cplx* lss;     // null, or L_ss of the separators solved by substitution (row-major) ...
  const cplx* lssc;    // ... and column-major packed (FactorArgs)
  const long long* lss_off;
  long long nlss;
  const int* flag;     // per RHS t: active iff (flag[t] != 0) == flag_on
  int flag_on;
  int sparse_rhs;      // host: RHS nonzero only on the transfer patches (forward plan fwd_sp)
  // sparse RHS only (else null): supernodes the forward touched; the others hold
  // z = 0 exactly, which the backward reads as 0 (X is not cleared)
  const unsigned char* sn_live;
  const cplx* B;       // right-hand sides (factor order), layout vm
  cplx* X;             // solutions (factor order), layout vm
  cplx* Y;             // scratch, layout vm
  VMap vm;
  int nw, nring;
};

// A member tile: up to 32 members of one class.
struct TileRec {
  long long cb;  // storage offset of (position 0, first member of the tile)
  int c;         // class
  int m;         // class member count = vector stride
  int t[32];     // RHS id of each tile member
};

// A tile group: tiles with the same member count M share every launch; the lane
// shape (R items x E element lanes x M members per warp) is set per launch.
struct TileArg {
  const TileRec* rec;
  int ntile;
  int M, E, R;
  unsigned magM = 0, magE = 0;  // ceil(2^32 / M), ceil(2^32 / E): x / d = umulhi(x, mag) for d > 1
};
inline unsigned div_magic(int d) { return d > 1 ? unsigned((0xffffffffull / unsigned(d)) + 1ull) : 0u; }
inline void tile_mags(TileArg& T) {
  T.magM = div_magic(T.M);
  T.magE = div_magic(T.E);
}

// One level of the level-synchronous sweeps: output items that are independent
// given the previous levels -- rows (supernode, row) / leaves (leaf, 0) forward,
// columns (supernode, column) backward.
// Forward pulls of member tiles on the FP64 tensor cores: the level's rows in blocks
// of up to 8 rows of one separator; per block the union of the rows' run segments by
// source supernode (columns [zmin, zmin + ulen)), each row's piece of it
// [lo, hi) with its values at vals[vb + z] (zero elsewhere: padding)
struct MmaSeg {
  int zmin, ulen;
  int lo[8], hi[8];
  long long vb[8];
};

struct SolveLevel {
  int nitem = 0;
  // member-tile forward pulls by DMMA (k_fwd_pull_mma): blocks (first item, rows,
  // first segment, segments)
  int nmblk = 0;
  int4* d_mblk = nullptr;
  MmaSeg* d_mseg = nullptr;
  double mma_fill = 0;  // padded / stored entries of the blocks
  int2* d_items = nullptr;
  int4* d_rec = nullptr;    // forward rows: (position, first segment, segment count, -)
  long avg_run = 0;         // forward: mean incoming run length
  long avg_diag = 0;        // forward: mean dense-inverse row length
  bool split_rows = false;  // backward pull: a CTA of 8 warps splits long row lists
  bool split_diag = false;  // backward diagonal: a CTA splits the inverse columns
  // backward split kernels: per columns-per-CTA R, the groups (supernode, first column)
  std::map<int, std::pair<int, int2*>> groups;
  // backward staged kernels: column chunks (supernode, j0, j1, -) of <= 32 columns
  int nchunk4 = 0;
  int4* d_chunks4 = nullptr;
  int cw_max = 0;
  bool one_chunk = false;   // every supernode of the level is one chunk (n <= the chunk width)
  // the level's separators (supernode, 0) for the substitution kernels
  int nsep = 0, nmax_sep = 0;
  int2* d_seps = nullptr;
};

struct SolvePlan {
  SolveLevel fwd_leaf;                 // leaves: band forward substitution
  std::vector<SolveLevel> fwd;         // separator rows by height (pull, then diag)
  SolveLevel fwd_leaf_sp;              // the same restricted to subtrees holding transfer-
  std::vector<SolveLevel> fwd_sp;      // patch nodes (steps >= 2; X cleared beforehand)
  bool has_sparse = false;
  SegRec* d_fseg = nullptr;            // segments referenced by fwd levels' records
  SegRec* d_fseg_sp = nullptr;         // live segments (active sources) for fwd_sp
  unsigned char* d_sn_live = nullptr;  // per supernode: in a subtree holding a patch node
  std::vector<SolveLevel> bwd;         // separator columns by depth (pull, then diag)
  SolveLevel bwd_leafcol;              // leaf columns: w = Dinv z - B^T x
  SolveLevel bwd_leaf;                 // leaves: band back-substitution
  std::vector<TileArg> groups;         // tile groups (E, R set per launch)
  std::vector<TileArg> sub;            // per group: its tiles split in 2-member sub-tiles
                                       // (ntile 0: none), for the levels with long rows
  long sub_run = 1L << 40;             // forward levels with mean run above: sub-tiles
                                       // (measured slower at config 4: HDDM_SUB_RUN opt-in)
  int sub_bwd_ctas = 128;              // backward staged levels that would launch fewer
                                       // CTAs use sub-tiles (measured -3 % at config 4)
  std::vector<TileRec> tiles;          // host copy of every tile
  std::vector<int> tile_group;         // group of each tile
  bool staged = true;                  // backward pulls through shared memory
  int pdl = 0;                         // programmatic dependent launch of the level chains:
                                       // 0 off, 1 every chain, 2 singleton-tile chains only
  // forward: CTA per row above these mean lengths (measured slower at config 4:
  // off by default, HDDM_CTA_RUN / HDDM_CTA_DIAG)
};

// one tile group's full solve (all levels) on one stream
void launch_solve_group(const SolveArgs& A, const SolvePlan& P, int g, cudaStream_t st);
int solve_launch_count(const SolvePlan& P, const SolveArgs& A);  // kernels of one solve over all tiles
void set_solve_skip(int mask, int only_tile);  // profiling aid (hddm_time_solve only)
// forward lane-shape override of the steady-state plan (tuning): which = 0/1 pulls of
// singleton / member tiles, 2/3 inverse rows; E = 0 restores the heuristic
void set_fwd_shape(int which, int level, int E);

// ------------------------------------------------------------------ factor
struct FactorArgs {
  const DevSn* sn;
  const DevBlk* blk;
  const int* row_first;
  const long long* row_off;
  const int* extadd;
  const int* aent_i;
  const int* aent_j;
  const cplx* aval;   // ncls x naent
  int naent;
  cplx* front;        // ncls x front_words
  long long front_words;
  cplx* vals;         // ncls x nvals
  long long nvals;
  cplx* lss;          // null, or ncls x nlss: diagonal blocks L_ss of the separators solved by
                      // substitution (packed lower, row-major) ...
  cplx* lssc;         // ... and column-major packed (column i: rows i+1..n-1)
  const long long* lss_off;  // per supernode: offset of its block, -1: applied as an inverse
  long long nlss;
  int* status;        // per class: 0 ok, 1 zero pivot
};

// fmax: largest front (own columns + update rows); the shared scratch is sized from it
void launch_factor_level(const FactorArgs& A, const int* d_nodes, int nnodes, int ncls, int fmax,
                         cudaStream_t st);
size_t factor_smem_limit();  // bytes of shared scratch available per CTA

// ------------------------------------------------------------------ DDM step
struct StepArgs {
  // geometry
  int n1, n2, nsub, nov, gnx, gny, wnx, wny, nw, nring, mcx, mcy;
  int npatch;            // structural union of the 8 transfer patches (window nodes)
  const int* pnode;
  const int* pmask;      // bit d: node lies in direction d's patch
  const int* xfer_pos;      // per (patch node, direction, stencil point): source position or -1
  const double* xfer_beta;  // ... and transfer_beta there
  const int4* xblk;         // transfer blocks: (class, first member slot, members, first patch node)
  int nxblk;
  const double* k2c;        // per class: window k^2 in factor order
  double ih2;
  const DevSub* sub;
  const cplx* sa;        // per-sub alpha arrays: a1n[wnx] ia1h[wnx] a2n[wny] ia2h[wny]
  int sa_stride;
  const double* wx;      // per-sub blend weights (nsub x wnx)
  const double* wy;      // (nsub x wny)
  const double* k2;      // global nodal k^2
  const int* perm;       // window node -> ... (perm[pos] = node)
  const int* pinv;       // node -> pos
  // state
  const cplx* f;         // global source/rhs of this sweep sequence
  const int* fany;       // per-sub: owned f has a nonzero
  int* zc;               // flags of this step (1 = zero/skipped)
  const int* zp1;
  const int* zp2;
  VMap vm;               // layout of B and the U vectors
  cplx* B;               // rhs (factor order)
  cplx* Ucur;            // this step's solutions (factor order)
  const cplx* Up1;       // previous step
  const cplx* Up2;       // two steps back
  cplx* asmb;            // assembled global field
  const int* colcov;     // per global column: up to 4 covering i (-1 pad)
  const int* rowcov;     // per global row: up to 4 covering j
  int step;
  // class membership and active lists
  const int* cls_ptr;
  const int* cls_mem;
  int* act_ptr;
  int* act_list;
  long long* counts;     // [0] solves, [1] skipped
  const int* owned;      // sharded runs (hddm_set_owned): subdomains this engine solves;
                         // the others are skipped here, their flags / solutions set by
                         // hddm_halo_unpack; null: every subdomain
};

void launch_fany(const StepArgs& A, cudaStream_t st);
void launch_flags(const StepArgs& A, int ncls, cudaStream_t st);
void launch_gather(const StepArgs& A, cudaStream_t st);
void launch_transfer(const StepArgs& A, cudaStream_t st);  // the 8-direction transfer pass alone
void launch_accumulate(const StepArgs& A, cudaStream_t st);

// per-RHS residual check of the local solve (refine's first pass,
// proj/src/sparse.cpp:268-292): rel[t] = ||B - A X|| / ||B||
struct CheckArgs {
  int nw, wnx, wny, gnx, nring;
  double ih2;
  const DevSub* sub;
  const cplx* sa;
  int sa_stride;
  const double* k2;
  const int* perm;
  const int* pinv;
  const int* zc;      // per RHS: 1 = inactive
  const int* only;    // if set: process RHS t only when only[t] != 0 (refinement re-checks)
  const int2* lpq;    // per factor position: window (p, q); p < 0 on the ring
  const int4* nbr;    // per factor position: S, W, E, N neighbour positions (-1: dropped)
  const double* k2c;  // per class: k^2 of its window in factor order
  const cplx* ctab;          // tabulated row coefficients (k_build_ctab) of the classes with
  const long long* ctab_off; // ctab_off[c] >= 0 (null: none)
  int nsub;
  VMap vm;
  const cplx* B;
  const unsigned char* bmask;  // per position: B may be nonzero (null: everywhere). Steps >= 2:
                               // the transfer-patch union (B is exactly 0 elsewhere)
  const cplx* X;
  double* part;      // nsub x nchunk x 2
  int nchunk;
  double* rel;       // per sub
  int* refine_flag;  // set when any rel > 1e-11
  double* max_rel;
};
void launch_build_ctab(const CheckArgs& A, int c, cplx* tab, cudaStream_t st);
void launch_check(const CheckArgs& A, cudaStream_t st);           // partials + per-RHS rel
void launch_check_partials(const CheckArgs& A, cudaStream_t st);  // partials only
struct RefineArgs;
// check partials, then per-RHS rel + refinement init (refine's first pass) in one kernel;
// `done` is a zeroed device counter
void launch_check_init(const CheckArgs& A, const RefineArgs& R, int* done, cudaStream_t st);
// the check of one tile group's members (queued on the group's stream after its
// solve) and, after all groups, the per-RHS statistics + refinement init
void launch_check_tiles(const CheckArgs& A, const TileArg& G, cudaStream_t st);
void launch_finish_init(const CheckArgs& A, const RefineArgs& R, int* done, cudaStream_t st);

// Iterative refinement on device (refine, proj/src/sparse.cpp:268-292): per RHS
// state after the first solve; corrections run inside a conditional WHILE graph
// node while any RHS still needs one.
struct RefineArgs {
  int nsub, ncls, nw, wnx, wny, gnx, nchunk;
  double ih2;
  const DevSub* sub;
  const cplx* sa;
  int sa_stride;
  const double* k2;
  const int* perm;
  const int* pinv;
  const int* zc;
  const int2* lpq;    // as CheckArgs
  const int4* nbr;
  const double* k2c;
  VMap vm;            // layout of B, X, R, C
  const cplx* B;
  cplx* X;
  cplx* R;            // residual vectors (correction right-hand sides)
  cplx* C;            // corrections
  const double* part; // check partials
  double* rel_cur;    // per RHS: last accepted relative residual
  int* need;          // per RHS: still refining
  int* ncorr;         // per RHS: corrections applied
  int* undo;          // per RHS: last correction to be undone
  int* any;           // device flag: some RHS needs a correction
  long long* nfix;    // total corrections applied (diagnostics)
  const int* cls_ptr;
  const int* cls_mem;
  int* act_ptr;
  int* act_list;
  unsigned long long cond;  // cudaGraphConditionalHandle (0: not in a graph)
};
void launch_refine_init(const RefineArgs& R, cudaStream_t st);   // after the first check
void launch_refine_prep(const RefineArgs& R, cudaStream_t st);   // act lists + residuals
void launch_refine_apply(const RefineArgs& R, cudaStream_t st);  // X += C
void launch_refine_decide(const RefineArgs& R, cudaStream_t st); // after the re-check
void launch_refine_undo(const RefineArgs& R, cudaStream_t st);

// ------------------------------------------------------------------ global
struct GlobalArgs {
  int gnx, gny;
  double ih2;
  const cplx* ga;   // a1n[gnx] ia1h[gnx] a2n[gny] ia2h[gny]
  const double* k2;
};
// out = L u (ring identity); if f != nullptr also partial sums of |f - out|^2
void launch_apply_global(const GlobalArgs& G, const cplx* u, cplx* out, const cplx* f,
                         double* part, cudaStream_t st);
// the same with u = U[*jp + du], out = O[*jp + dout] (device-resident Krylov index j)
void launch_apply_global_ind(const GlobalArgs& G, cplx* const* U, int du, cplx* const* O, int dout,
                             const int* jp, cudaStream_t st);
int reduce_blocks();  // number of partials the reduction kernels produce

// deterministic reductions / BLAS-1 over n complex
void launch_nrm2_part(const cplx* v, long long n, double* part, cudaStream_t st);
void launch_dot_part(const cplx* a, const cplx* b, long long n, double* part, cudaStream_t st);
// sum partials (reduce_blocks() of them, stride 1 or 2 doubles) into out
void launch_finish_sum(const double* part, int ncomp, double* out, cudaStream_t st);

}  // namespace hddm
