// state.h -- internal definition of qc_state and the cached plans (shared by
// api.cu and dist.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "qc_internal.h"

namespace qc {

struct PlanEntry {
  std::vector<qc_gate> ops;          // exact copy (collision check)
  std::vector<uint8_t> mkey;         // referenced generic gates' contents (collision check)
  std::vector<int> layout_in, layout_out;
  std::vector<PassDesc> passes;
  void* d_blob = nullptr;
  int64_t fused_gates = 0;
  std::shared_ptr<FusedPlan> ir;     // kept for JIT specialisation
  std::vector<JitKernel> jit;
  int jit_state = 0;                 // 0 not tried, 1 built, -1 failed
  QcTmap tmap{};                     // row tensor map (gather4 / scatter4 path)
  std::vector<QcTmap> tmaps;         // per-pass box tensor maps (PassDesc g4 == 2; empty otherwise)
  // plans spanning shards (dist.cu, QC_OPT_EXCHANGE 2 / 3): rank bits in the plan
  uint64_t group_mask = 0;           // plan bits that are rank bits (pair / group plans); 0: none
  QcTmap tmap_peer{};                // the partner's buffer (P2P): row tensor map ...
  std::vector<QcTmap> tmaps_peer;    // ... and per-pass box tensor maps
  // loopback pair segments: tensor maps over each virtual rank's own shard
  // (nl bits at that shard's base), so the loopback runs the P2P code path
  // -- separate buffers, addr_bits 0 -- with only the pointers local
  std::vector<QcTmap> vr_row;               // [rank]
  std::vector<std::vector<QcTmap>> vr_box;  // [rank][pass]
  bool dbl = true;
  int64_t relabels = 0;
  int uses = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int ctas = 0;
  int tile_bits = 0;
  std::vector<int> perm;             // remap: data of physical bit p ends at perm[p]
  double flops_per_amp = 0;          // plan_flops_per_amp
  ~PlanEntry() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (d_blob) cudaFree(d_blob);
  }
};


// Generic gates of qc_run_circuit_ex / qc_apply_mgate, copied (matrix
// included) so plans never point into caller memory.
struct MGate {
  int n_ctrl = 0, n_targ = 0;
  int qubits[QC_MGATE_MAX_QUBITS] = {};
  uint32_t ctrl_state = 0;
  std::vector<cd> m;  // row-major 2^n_targ x 2^n_targ
};
using MTable = std::vector<MGate>;
// Content bytes of the gates an op list references (plan-cache key / check).
std::vector<uint8_t> mtable_key(const qc_gate* ops, size_t n_ops, const MTable* mt);
// Logical qubits of an op (controls first), and its non-diagonal targets.
int op_qubits(const qc_gate& g, const MTable* mt, int* out);
uint64_t op_nondiag_mask(const qc_gate& g, const MTable* mt);

struct DistPlan;   // dist.cu
struct DistCache;  // dist.cu

// api.cu helpers shared with dist.cu
qc_status fail(qc_status st, const char* fmt, ...);
qc_status cuda_fail(qc_state* s, int e, const char* what);
PGate lower(const qc_gate& g, const int* layout, const MTable* mt = nullptr);
qc_status validate_gate(int n, const qc_gate& g, size_t idx, const MTable* mt = nullptr);
uint64_t hash_ops(const qc_gate* ops, size_t n, const int* layout, int nq, uint64_t salt);
qc_status build_fused_entry(qc_state* s, const std::vector<PGate>& gates, int n_plan, uint64_t local_mask,
                            PlanEntry* e, void* tmap_base = nullptr, int tmap_bits = 0, bool remap = false,
                            uint64_t group_mask = 0, void* peer_base = nullptr);
int enqueue_entry(qc_state* s, PlanEntry* e, cudaStream_t st, void* base, uint64_t rank_bits,
                  uint64_t addr_bits);
uint64_t pass_tile_set(const PassDesc& d);  // a pass's tile bit set (row bits + hi bits)
// One pass of an entry with explicit buffers (pair segments: halves in two buffers).
int launch_pass(qc_state* s, PlanEntry* e, size_t i, const PassDesc& pd, void* base, const QcTmapSet& tms,
                cudaStream_t st);
qc_status maybe_jit(qc_state* s, PlanEntry* e);
qc_status ensure_fused_configured(qc_state* s);
extern const int kArity[16];
extern const int kNctrl[16];

// dist.cu
qc_status run_dist(qc_state* s, const qc_gate* ops, size_t n_ops, const MTable* mt = nullptr);
qc_status dist_canonicalize(qc_state* s);
qc_status dist_exchange(qc_state* s, int g, int l);
qc_status nccl_create_comm(qc_state* s, const void* unique_id);
qc_status nccl_get_unique_id(void* out128);
qc_status nccl_allreduce_sum(qc_state* s, double* host_value);
void nccl_destroy(qc_state* s);
void dist_release(qc_state* s);  // drop sharded plans + communicator
qc_status dist_schedule_dry(int n, int world, int relabel, const qc_gate* ops, size_t n_ops,
                            std::vector<int>& out, std::vector<int>& layout_out, const MTable* mt = nullptr,
                            int xmode = 0);
struct GroupSplit {
  uint64_t tile0 = 0, count = 0;  // this rank's tile range of the pass
  int j = 0;                      // rank bits in the tile
  int owner[8] = {};              // rank holding sub-tile h (h < 2^j)
};
GroupSplit group_split(int nl, int p, uint64_t T, uint64_t n_tiles, int r);
struct ExchangeRun {
  uint64_t offset;  // amplitudes, within the shard
  uint64_t count;
};
// The part of rank `rank`'s shard that an exchange of global bit g with local
// bit l sends (and receives into): local indices y with bit l == 1 - bit g.
std::vector<ExchangeRun> exchange_runs(int n_loc, int rank, int g, int l, int* partner);

}  // namespace qc

struct qc_state {
  int n = 0;
  qc_precision prec = QC_COMPLEX128;
  bool dbl = true;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* d = nullptr;
  bool own_mem = false;
  size_t bytes = 0;
  int layout[64];
  bool failed = false;
  // options
  int fusion = 1, relabel = 1, use_graph = 1, tile_bits = 0, ctas = 0, block_fusion = 1, jit = 1;
  int row_bits = 0, tma_mode = 0;
  int remap = 1;  // QC_OPT_REMAP
  std::string jit_error;
  // stats
  int64_t last_gates = 0, last_passes = 0, last_launches = 0, last_relabels = 0;
  int last_graph = 0, last_k = 0;
  int64_t last_blocks = 0;
  int last_jit = 0;
  double last_flops_per_amp = 0;
  // plan cache
  std::unordered_map<uint64_t, std::unique_ptr<qc::PlanEntry>> plans;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cstream = nullptr;    // qc_state_readwrite: upload stream (D2H stays on `stream`)
  cudaEvent_t cev[2] = {};
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  double* d_partial = nullptr;
  // sharded state: physical bits >= n_loc are rank bits
  int dist = 0;       // 0: single GPU; 1: loopback (all ranks' shards in this buffer); 2: NCCL
  int world = 1, rank = 0, n_loc = 0;
  void* nccl_comm = nullptr;
  void* d_xstage = nullptr;          // exchange staging: two chunks (ping-pong)
  size_t xstage_bytes = 0;
  int xmode = 0;                     // QC_OPT_EXCHANGE: 0 NCCL send/recv, 1 P2P swap kernel, 2 pair passes
  cudaStream_t xstream = nullptr;    // NCCL exchange stream (copies stay on `stream`)
  cudaEvent_t xev[5] = {};           // start, recv_done[2], copy_done[2]
  std::vector<void*> peers;          // P2P: every rank's state buffer, IPC-mapped (own: d)
  int* d_token = nullptr;            // P2P: pairwise barrier token (2 ints)
  int64_t last_exchanges = 0;
  int64_t last_pair_segments = 0;
  qc::DistCache* dcache = nullptr;  // sharded plans (owned by dist.cu)
  ~qc_state();
};

