// Host side of the dataflow solve plan (dag.cuh, dag_plan.cu).
#pragma once

#include <vector>

#include "dag.cuh"
#include "hddm_internal.h"

namespace hddm {

struct DagTileIn {  // a member tile as the engine cuts it
  long long cb;
  int c, m, M;
  int t[kDagMaxM];
};

struct DagPlanHost {
  std::vector<DagSn> sn;
  std::vector<int> row_first, row_dpos, col_off;
  std::vector<long long> row_boff;
  struct Dec {
    int hb = 0, G = 0;
    std::vector<DagUnit> unit;
    std::vector<DagLv> lv;
    int M = 0;
    std::vector<int> lsn, lsr, lrow, row_slot, in_ptr, in_ref, ext_src, ext_tgt, unit_of;
    std::vector<DagSn> lvsn;
    std::vector<int> lrm;  // 4 ints per level row
    std::vector<int> lrx, xe;
    std::vector<DagChunk> ch;
    std::vector<int> cmeta;
    std::vector<unsigned char> in_live;
    std::vector<DagExt> ext;
    long long smem_need = 0;           // bytes of shared memory a CTA needs (after finalize)
    // per unit: stage the factor values when they fit next to the vectors; returns the
    // shared memory needed, or a huge value when a subtree unit cannot stage them
    long long finalize(int M, long long budget, const Symbolic& Y);
  };
  std::vector<Dec> dec;
  std::vector<DagTile> tile;
  std::vector<DagTask> task;
  long long nP = 0;      // partial slots (complex)
  long long smem_bytes = 0;
};

int dag_smem_budget();
// live_sn: per supernode, its subtree holds transfer-patch nodes (steps >= 2)
void build_dag_plan(const Symbolic& Y, const std::vector<char>& live_sn,
                    const std::vector<DagTileIn>& tiles, DagPlanHost& P);

}  // namespace hddm
