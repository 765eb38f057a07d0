// Drop-in replacement of the reference's proj/include/helmddm/ddm.hpp.
//
// The public surface is the reference's, unchanged (DdmConfig, StepRecord,
// DdmStats, OpClassInfo and DdmEngine with the same members, argument meaning,
// return types and exceptions -- ddm.hpp:15-109); only the private state differs:
// the engine is the B200 one behind the C-ABI of libhddm.so (include/hddm.h).
// A maintainer switches the reference to the GPU path by
//   * putting this directory before proj/include on the include path,
//   * compiling paper_1807_04180_b200/dropin/ddm_b200.cpp instead of src/ddm.cpp,
//   * linking libhddm.so;
// every other reference source -- cli.cpp, krylov.cpp (the host fgmres drives the
// GPU apply_global / precondition through its LinearOp callbacks), config.cpp,
// io.cpp, the tests -- compiles unchanged.
#pragma once

#include <memory>

#include "helmddm/discretize.hpp"
#include "helmddm/medium.hpp"
#include "helmddm/partition.hpp"
#include "helmddm/sparse.hpp"
#include "helmddm/threads.hpp"
#include "helmddm/transfer.hpp"
#include "helmddm/types.hpp"

struct hddm_engine;

namespace helmddm {

struct DdmConfig {
  GridSpec grid;
  MediumModel medium;
  double c_sigma = 25.0;
  double sigma0 = 0;      // > 0 overrides the c_sigma-derived plateau
  bool force_lu = false;  // accepted; the GPU path has only the LDL^T backend
  int threads = 1;        // accepted; the GPU replaces the worker pool
};

struct StepRecord {
  int step = 0;
  double relres = 0;
  double wall_ms = 0;
};

struct DdmStats {
  int steps = 0;
  long solves = 0;
  long skipped = 0;
  double relres = -1;
  bool converged = false;
  double factor_ms = 0;
  double sweep_ms = 0;
  std::vector<StepRecord> history;
};

struct OpClassInfo {
  int members = 0;
  const char* backend = "";
  size_t factor_nnz = 0;
  double probe_relres = 0;
};

/// The reference's additive overlapping DDM engine (ddm.hpp:47-109), on one B200.
class DdmEngine {
 public:
  explicit DdmEngine(const DdmConfig& cfg);
  ~DdmEngine();
  DdmEngine(const DdmEngine&) = delete;
  DdmEngine& operator=(const DdmEngine&) = delete;

  const Partition& partition() const { return part_; }
  const GridSpec& grid() const { return part_.g; }
  const DiscreteOperator& global_op() const { return gop_; }
  double sigma0() const { return sigma0_; }
  size_t n_global() const { return gop_.k2.size(); }
  double factor_ms() const { return factor_ms_; }
  std::vector<OpClassInfo> class_info() const;

  void apply_global(const Complex* u, Complex* out) const;

  FieldGrid solve_iterative(const std::vector<Complex>& f, double tol, int max_steps,
                            DdmStats& stats, int check_every = 1);

  void precondition(const Complex* r, Complex* z, int ksteps, DdmStats& stats);

 private:
  DdmConfig cfg_;
  Partition part_;
  double sigma0_ = 0;
  double factor_ms_ = 0;
  DiscreteOperator gop_;  // the global operator, built by the reference's own code
  hddm_engine* eng_ = nullptr;
};

}  // namespace helmddm
