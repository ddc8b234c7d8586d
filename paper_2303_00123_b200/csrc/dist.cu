// dist.cu -- the sharded state (north star "shards the vector
// across the B200s by its top log2(P) qubits and remaps global to local qubits
// through NCCL pairwise send/recv").
//
// A state of n qubits over P = 2^p ranks keeps 2^{n_loc} = 2^{n-p} amplitudes
// per rank; physical bits >= n_loc are rank bits.  Every gate is still the
// eq:kron operator; on a shard:
//   * a gate whose non-diagonal targets are local runs in the fused engine on
//     the shard; controls / diagonal bits on rank bits are per-rank constants
//     (PassDesc::rank_bits is OR-ed into every tile's base index);
//   * a non-diagonal target on a rank bit g first swaps g with a local bit l
//     ("qubit-swap exchange"): rank r and its partner r ^ 2^{g-n_loc} trade
//     the local half where bit l != their bit g; afterwards the logical qubits
//     at g and l have exchanged physical positions (layout update).
// The schedule is computed identically on every rank (host, deterministic):
// the local victim is the qubit whose next non-diagonal use is farthest away
// (Belady); if it is not already at the exchange slot l = n_loc-1 a physical
// SWAP of the two local bits is inserted into the preceding fused segment,
// so every exchange moves ONE contiguous half shard per direction.
//
// Backends: NCCL (one process per GPU; libnccl dlopen'ed, grouped chunked
// ncclSend/ncclRecv through a staging buffer, stream-ordered) and loopback
// (all P shards of one process in one buffer on one GPU; the exchange swaps
// the same runs in place) -- the latter exercises the whole sharded path on a
// single GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <bit>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "state.h"

qc_state::~qc_state() {}

namespace qc {

struct DistPlan {
  std::vector<qc_gate> ops;
  std::vector<uint8_t> mkey;  // referenced generic gates' contents
  std::vector<int> layout_in, layout_out;
  struct Step {
    int kind = 0;  // 0: fused local segment, 1: exchange, 2: pair segment on rank bit g (QC_OPT_EXCHANGE 2),
                   // 3: the whole circuit as one plan over all n bits (QC_OPT_EXCHANGE 3)
    int g = -1, l = -1;
    bool restore = false;  // exchange that undoes the schedule's permutation at the end
    std::unique_ptr<PlanEntry> seg;
  };
  std::vector<Step> steps;
  int64_t exchanges = 0, relabels = 0, passes = 0, pair_segments = 0;
  int64_t restore_exchanges = 0;  // of `exchanges`: undoing the schedule's permutation at the end
  int uses = 0;
};

struct DistCache {
  std::unordered_map<uint64_t, std::unique_ptr<DistPlan>> plans;
};

namespace {

// ------------------------------------------------------------------ NCCL
typedef struct {
  char internal[128];
} QcNcclId;
enum { kNcclUint8 = 1, kNcclFloat64 = 8, kNcclSum = 0 };
struct Nccl {
  int (*get_unique_id)(QcNcclId*) = nullptr;
  int (*comm_init_rank)(void**, int, QcNcclId, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("QC_NCCL_LIB");
    const char* names[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if (nm && (h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return;
#define QC_NSYM(f, s) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, s))
    QC_NSYM(get_unique_id, "ncclGetUniqueId");
    QC_NSYM(comm_init_rank, "ncclCommInitRank");
    QC_NSYM(comm_destroy, "ncclCommDestroy");
    QC_NSYM(send, "ncclSend");
    QC_NSYM(recv, "ncclRecv");
    QC_NSYM(group_start, "ncclGroupStart");
    QC_NSYM(group_end, "ncclGroupEnd");
    QC_NSYM(all_reduce, "ncclAllReduce");
    QC_NSYM(all_gather, "ncclAllGather");
    QC_NSYM(error_string, "ncclGetErrorString");
#undef QC_NSYM
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.send && n.recv && n.group_start &&
           n.group_end && n.all_reduce && n.all_gather;
  });
  return n;
}

qc_status nccl_fail(qc_state* s, int r, const char* what) {
  if (s) s->failed = true;
  return fail(QC_ERR_NCCL, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "nccl error");
}


}  // namespace

std::vector<ExchangeRun> exchange_runs(int n_loc, int rank, int g, int l, int* partner) {
  const int gb = g - n_loc;
  if (partner) *partner = rank ^ (1 << gb);
  const uint64_t mybit = (uint64_t)((rank >> gb) & 1);
  const uint64_t want = 1 - mybit;  // bit l of the local indices that are traded
  std::vector<ExchangeRun> runs;
  const uint64_t run = 1ull << l;
  const uint64_t nruns = 1ull << (n_loc - 1 - l);
  for (uint64_t k = 0; k < nruns; ++k) runs.push_back({k * 2 * run + want * run, run});
  return runs;
}

qc_status nccl_create_comm(qc_state* s, const void* unique_id) {
  Nccl& N = nccl();
  if (!N.ok) return fail(QC_ERR_NCCL, "libnccl.so.2 not found (set QC_NCCL_LIB)");
  QcNcclId id;
  std::memcpy(&id, unique_id, sizeof id);
  const int r = N.comm_init_rank(&s->nccl_comm, s->world, id, s->rank);
  if (r) return nccl_fail(s, r, "ncclCommInitRank");
  return QC_OK;
}

qc_status nccl_get_unique_id(void* out128) {
  Nccl& N = nccl();
  if (!N.ok) return fail(QC_ERR_NCCL, "libnccl.so.2 not found (set QC_NCCL_LIB)");
  QcNcclId id;
  const int r = N.get_unique_id(&id);
  if (r) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
  return QC_OK;
}

void dist_release(qc_state* s) {
  delete s->dcache;
  s->dcache = nullptr;
  for (int r = 0; r < (int)s->peers.size(); ++r)
    if (r != s->rank && s->peers[r]) cudaIpcCloseMemHandle(s->peers[r]);
  s->peers.clear();
  nccl_destroy(s);
}

void nccl_destroy(qc_state* s) {
  if (s->nccl_comm && nccl().ok) nccl().comm_destroy(s->nccl_comm);
  s->nccl_comm = nullptr;
}

qc_status nccl_allreduce_sum(qc_state* s, double* host_value) {
  Nccl& N = nccl();
  double* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(double), s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaMallocAsync");
  cudaMemcpyAsync(d, host_value, sizeof(double), cudaMemcpyHostToDevice, s->stream);
  const int r = N.all_reduce(d, d, 1, kNcclFloat64, kNcclSum, s->nccl_comm, s->stream);
  if (r) return nccl_fail(s, r, "ncclAllReduce");
  cudaMemcpyAsync(host_value, d, sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  cudaFreeAsync(d, s->stream);
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamSynchronize");
  return QC_OK;
}

namespace {

// Staging (bytes), the exchange stream and its events, created on first use.
qc_status ensure_xresources(qc_state* s, size_t bytes) {
  if (s->xstage_bytes < bytes) {
    if (s->d_xstage) cudaFree(s->d_xstage);
    s->d_xstage = nullptr;
    s->xstage_bytes = 0;
    cudaError_t e = cudaMalloc(&s->d_xstage, bytes);
    if (e != cudaSuccess) return fail(QC_ERR_OUT_OF_MEMORY, "exchange staging (%zu B)", bytes);
    s->xstage_bytes = bytes;
  }
  if (!s->xstream) {
    cudaError_t e = cudaStreamCreateWithFlags(&s->xstream, cudaStreamNonBlocking);
    for (int i = 0; i < 5 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&s->xev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(s, e, "exchange stream");
  }
  return QC_OK;
}

// Collective, once per state: all-gather every rank's CUDA IPC handle of its
// state buffer over NCCL and map the other ranks' buffers (peer access over
// NVLink; cudaIpcMemLazyEnablePeerAccess).
qc_status ensure_peers(qc_state* s) {
  if (!s->peers.empty()) return QC_OK;
  Nccl& N = nccl();
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, s->d);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaIpcGetMemHandle");
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  std::vector<cudaIpcMemHandle_t> all((size_t)s->world);
  char* d = nullptr;
  e = cudaMalloc(&d, hb * (size_t)(s->world + 1));
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaMalloc (IPC handles)");
  e = cudaMemcpyAsync(d, &h, hb, cudaMemcpyHostToDevice, s->stream);
  int r = e == cudaSuccess ? N.all_gather(d, d + hb, hb, kNcclUint8, s->nccl_comm, s->stream) : 0;
  if (e == cudaSuccess && !r) e = cudaMemcpyAsync(all.data(), d + hb, hb * s->world, cudaMemcpyDeviceToHost, s->stream);
  if (e == cudaSuccess && !r) e = cudaStreamSynchronize(s->stream);
  cudaFree(d);
  if (r) return nccl_fail(s, r, "ncclAllGather (IPC handles)");
  if (e != cudaSuccess) return cuda_fail(s, e, "IPC handle exchange");
  s->peers.assign((size_t)s->world, nullptr);
  for (int q = 0; q < s->world; ++q) {
    if (q == s->rank) {
      s->peers[q] = s->d;
      continue;
    }
    e = cudaIpcOpenMemHandle(&s->peers[q], all[q], cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      s->peers.clear();
      return cuda_fail(s, e, "cudaIpcOpenMemHandle");
    }
  }
  if (!s->d_token) {
    e = cudaMalloc(&s->d_token, 2 * sizeof(int));
    if (e != cudaSuccess) return cuda_fail(s, e, "cudaMalloc (token)");
  }
  return QC_OK;
}

// Stream-ordered pairwise barrier: a 1-int NCCL send/recv with the partner
// completes only after the partner has enqueued (and its stream reached) the
// matching call, i.e. after every earlier kernel on the partner's stream.
qc_status pair_barrier(qc_state* s, int partner) {
  Nccl& N = nccl();
  int r = N.group_start();
  if (!r) r = N.send(s->d_token, 1, kNcclUint8, partner, s->nccl_comm, s->stream);
  if (!r) r = N.recv(s->d_token + 1, 1, kNcclUint8, partner, s->nccl_comm, s->stream);
  const int r2 = N.group_end();
  if (r || r2) return nccl_fail(s, r ? r : r2, "pair barrier");
  return QC_OK;
}

// P2P exchange: the pair swaps my run with the partner's matching run in
// place -- the lower rank the first half of every run, the upper rank the
// second half -- with one kernel reading and writing both buffers (the
// partner's through its IPC mapping, i.e. NVLink loads and stores).
qc_status p2p_exchange(qc_state* s, int g, int l) {
  qc_status st = ensure_peers(s);
  if (st != QC_OK) return st;
  const size_t ab = s->dbl ? 16 : 8;
  int partner;
  const auto mine = exchange_runs(s->n_loc, s->rank, g, l, &partner);
  const auto theirs = exchange_runs(s->n_loc, partner, g, l, nullptr);
  st = pair_barrier(s, partner);  // partner's earlier passes are done with its buffer
  if (st != QC_OK) return st;
  const bool lower = s->rank < partner;
  for (size_t k = 0; k < mine.size(); ++k) {
    const size_t bytes = mine[k].count * ab, half = (bytes / 2) & ~(size_t)15;
    const size_t off = lower ? 0 : half, len = lower ? half : bytes - half;
    char* a = (char*)s->d + mine[k].offset * ab + off;
    char* b = (char*)s->peers[partner] + theirs[k].offset * ab + off;
    const int e = launch_swap_regions(a, b, len, s->stream);
    if (e) return cuda_fail(s, e, "P2P exchange kernel");
  }
  return pair_barrier(s, partner);  // the partner's half of the swap is done too
}

}  // namespace

// Swap physical rank bit g with local bit l (stream-ordered).
qc_status dist_exchange(qc_state* s, int g, int l) {
  const size_t ab = s->dbl ? 16 : 8;
  if (s->dist == 1) {  // loopback: rank r's shard is [r << n_loc, (r+1) << n_loc) of one buffer
    for (int r = 0; r < s->world; ++r) {
      int partner;
      const auto mine = exchange_runs(s->n_loc, r, g, l, &partner);
      if (partner < r) continue;  // each pair once
      const auto theirs = exchange_runs(s->n_loc, partner, g, l, nullptr);
      for (size_t k = 0; k < mine.size(); ++k) {
        char* a = (char*)s->d + (((uint64_t)r << s->n_loc) + mine[k].offset) * ab;
        char* b = (char*)s->d + (((uint64_t)partner << s->n_loc) + theirs[k].offset) * ab;
        const int e = launch_swap_regions(a, b, mine[k].count * ab, s->stream);
        if (e) return cuda_fail(s, e, "loopback exchange");
      }
    }
    return QC_OK;
  }
  if (s->xmode >= 1) return p2p_exchange(s, g, l);  // (2: a gate needing two rank bits at once)
  // NCCL: send my runs to the partner, receive its runs into the same places.
  // Chunks alternate between two staging buffers: chunk i's send/recv runs on
  // the exchange stream while chunk i-1's copy into place runs on the state's
  // stream (the copy of chunk i waits for its recv; the recv of chunk i+2
  // into the same buffer waits for that copy).
  Nccl& N = nccl();
  int partner;
  const auto runs = exchange_runs(s->n_loc, s->rank, g, l, &partner);
  const size_t chunk_max = 256ull << 20;
  qc_status st = ensure_xresources(s, 2 * chunk_max);
  if (st != QC_OK) return st;
  cudaStream_t xs = s->xstream;
  cudaEvent_t start = s->xev[0], recv_done[2] = {s->xev[1], s->xev[2]}, copy_done[2] = {s->xev[3], s->xev[4]};
  cudaError_t e = cudaEventRecord(start, s->stream);  // the exchange follows the state's prior work
  if (e == cudaSuccess) e = cudaStreamWaitEvent(xs, start, 0);
  if (e != cudaSuccess) return cuda_fail(s, e, "exchange ordering");
  size_t i = 0;
  for (const auto& run : runs) {
    const size_t bytes = run.count * ab;
    char* base = (char*)s->d + run.offset * ab;
    for (size_t off = 0; off < bytes; off += chunk_max, ++i) {
      const size_t m = std::min(chunk_max, bytes - off);
      const int b = (int)(i & 1);
      char* stage = (char*)s->d_xstage + b * chunk_max;
      if (i >= 2 && (e = cudaStreamWaitEvent(xs, copy_done[b], 0)) != cudaSuccess)
        return cuda_fail(s, e, "exchange ordering");
      int r = N.group_start();
      if (!r) r = N.send(base + off, m, kNcclUint8, partner, s->nccl_comm, xs);
      if (!r) r = N.recv(stage, m, kNcclUint8, partner, s->nccl_comm, xs);
      const int r2 = N.group_end();
      if (r || r2) return nccl_fail(s, r ? r : r2, "exchange send/recv");
      e = cudaEventRecord(recv_done[b], xs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, recv_done[b], 0);
      if (e == cudaSuccess) e = cudaMemcpyAsync(base + off, stage, m, cudaMemcpyDeviceToDevice, s->stream);
      if (e == cudaSuccess) e = cudaEventRecord(copy_done[b], s->stream);
      if (e != cudaSuccess) return cuda_fail(s, e, "exchange copy");
    }
  }
  return QC_OK;
}

namespace {

// Build the exchange / segment schedule for an op list from the state's layout.
// dry_run: schedule only (no device work; segments record their gate count).
// (masks are 64-bit: logical qubits reach 39; a 32-bit shift would alias q and q-32)
qc_status build_dist_plan(qc_state* s, const qc_gate* ops, size_t n_ops, DistPlan* P, const MTable* mt,
                          bool dry_run = false) {
  const int n = s->n, nl = s->n_loc;
  const int L = nl - 1;  // exchange slot: the top local bit (one contiguous half per direction)
  int lay[64], inv[64], rel[64];
  std::memcpy(lay, s->layout, sizeof(int) * n);
  std::memcpy(rel, s->layout, sizeof(int) * n);  // the layout after the SWAP relabels only
  for (int q = 0; q < n; ++q) inv[lay[q]] = q;
  if (s->xmode == 3) {
    // Group plan: the circuit is planned ONCE over all n bits, exactly like a
    // single-GPU state; a tile may hold rank bits, its sub-tiles then live in
    // several shards (PassDesc::grp).  No exchanges; the plan restores its
    // layout (remap) so only the SWAP relabels change it.
    std::vector<PGate> gates;
    for (size_t i = 0; i < n_ops; ++i) {
      const qc_gate& op = ops[i];
      if (op.op == QC_SWAP && s->relabel) {
        std::swap(lay[op.qubits[0]], lay[op.qubits[1]]);
        P->relabels++;
        continue;
      }
      gates.push_back(lower(op, lay, mt));
    }
    DistPlan::Step st;
    st.kind = 3;
    st.seg = std::make_unique<PlanEntry>();
    if (!gates.empty() && !dry_run) {
      const size_t shard_bytes = (size_t)(s->dbl ? 16 : 8) << nl;
      if (s->dist == 2) {
        const qc_status r = ensure_peers(s);  // collective (same point of the schedule on every rank)
        if (r != QC_OK) return r;
      }
      auto buf_of = [&](int q) -> void* {
        return s->dist == 1 ? (void*)((char*)s->d + (size_t)q * shard_bytes) : s->peers[(size_t)q];
      };
      const uint64_t rank_mask = ((n >= 64 ? ~0ull : (1ull << n) - 1)) & ~((1ull << nl) - 1);
      PlanEntry* e = st.seg.get();
      qc_status r = build_fused_entry(s, gates, n, ~0ull, e, buf_of(0), nl, s->remap != 0, rank_mask, buf_of(1));
      // tensor maps over every rank's shard (nl bits at its base)
      e->vr_row.assign((size_t)s->world, QcTmap{});
      e->vr_box.assign((size_t)s->world, std::vector<QcTmap>(e->passes.size(), QcTmap{}));
      for (int v = 0; v < s->world && r == QC_OK; ++v) {
        if (!e->passes.empty() && e->passes[0].g4 && !make_row_tmap(buf_of(v), nl, e->passes[0].rb, s->dbl, &e->vr_row[(size_t)v]))
          r = fail(QC_ERR_CUDA, "shard row tensor map");
        for (size_t i = 0; i < e->passes.size() && r == QC_OK; ++i) {
          PassDesc tmp = e->passes[i];
          if (e->passes[i].g4 == 2 &&
              !make_box_tmap(buf_of(v), nl, s->dbl, pass_tile_set(e->passes[i]) & ~rank_mask, &e->vr_box[(size_t)v][i],
                             &tmp))
            r = fail(QC_ERR_CUDA, "shard box tensor map");
        }
      }
      if (r != QC_OK) return r;
      if (!e->perm.empty())  // remap swaps moved physical bits: the layout follows the data
        for (int q = 0; q < n; ++q) lay[q] = e->perm[lay[q]];
      P->passes += (int64_t)e->passes.size();
      for (const PassDesc& pd : e->passes) P->pair_segments += pd.grp ? 1 : 0;  // passes spanning shards
    }
    st.seg->fused_gates = (int64_t)gates.size();
    if (!gates.empty()) P->steps.push_back(std::move(st));
    P->layout_out.assign(lay, lay + n);
    return QC_OK;
  }
  // next non-diagonal use of each logical qubit after op i (Belady)
  std::vector<std::vector<int>> uses(n);
  for (size_t i = 0; i < n_ops; ++i) {
    if (ops[i].op == QC_SWAP && s->relabel) continue;
    const uint64_t m = op_nondiag_mask(ops[i], mt);
    for (int q = 0; q < n; ++q)
      if (m & (1ull << q)) uses[q].push_back((int)i);
  }
  auto next_use = [&](int q, size_t i) -> long {
    auto it = std::upper_bound(uses[q].begin(), uses[q].end(), (int)i);
    return it == uses[q].end() ? (long)1 << 40 : (long)*it;
  };
  std::vector<PGate> seg;
  int seg_pair = -1;  // >= 0: the current segment is a pair segment on this rank bit
  auto flush = [&]() -> qc_status {
    if (seg.empty()) {
      seg_pair = -1;
      return QC_OK;
    }
    DistPlan::Step st;
    st.kind = seg_pair >= 0 ? 2 : 0;
    st.g = seg_pair;
    st.seg = std::make_unique<PlanEntry>();
    if (dry_run) {
      st.seg->fused_gates = (int64_t)seg.size();
      P->steps.push_back(std::move(st));
      seg.clear();
      seg_pair = -1;
      return QC_OK;
    }
    qc_status r;
    if (seg_pair < 0) {
      const uint64_t local_mask = (1ull << nl) - 1;
      // remap on: the plan ends in the layout it started from (restore passes),
      // so the exchange slot keeps the qubit the preceding SWAP2 put there
      r = build_fused_entry(s, seg, nl, local_mask, st.seg.get(), s->d, s->dist == 1 ? n : nl, s->remap != 0);
    } else {
      // pair segment: plan space = the nl local bits + the rank bit seg_pair
      // relabelled to plan bit nl (the other rank bits stay constants)
      for (PGate& pg : seg)
        if (seg_pair != nl) pgate_swap_bits(pg, nl, seg_pair);
      void* peer = nullptr;
      const size_t shard_bytes = (size_t)(s->dbl ? 16 : 8) << nl;
      if (s->dist == 2) {
        r = ensure_peers(s);  // collective (same point of the schedule on every rank)
        if (r != QC_OK) return r;
        peer = s->peers[(size_t)(s->rank ^ (1 << (seg_pair - nl)))];
      } else {
        peer = (char*)s->d + shard_bytes;  // loopback: shard 1 stands in for "a peer" (maps below)
      }
      // tensor maps over nl bits of one shard (the loopback too: it then
      // addresses every shard as its own buffer, like the IPC-mapped peers)
      r = build_fused_entry(s, seg, nl + 1, (2ull << nl) - 1, st.seg.get(), s->d, nl, s->remap != 0, 1ull << nl,
                            peer);
      if (r == QC_OK && s->dist == 1) {
        PlanEntry* e = st.seg.get();
        e->vr_row.assign((size_t)s->world, QcTmap{});
        e->vr_box.assign((size_t)s->world, std::vector<QcTmap>(e->passes.size(), QcTmap{}));
        for (int v = 0; v < s->world && r == QC_OK; ++v) {
          char* base = (char*)s->d + (size_t)v * shard_bytes;
          if (!e->passes.empty() && e->passes[0].g4 && !make_row_tmap(base, nl, e->passes[0].rb, s->dbl, &e->vr_row[(size_t)v]))
            r = fail(QC_ERR_CUDA, "loopback shard row tensor map");
          for (size_t i = 0; i < e->passes.size() && r == QC_OK; ++i) {
            PassDesc tmp = e->passes[i];
            if (e->passes[i].g4 == 2 &&
                !make_box_tmap(base, nl, s->dbl, pass_tile_set(e->passes[i]) & ~(1ull << nl),
                               &e->vr_box[(size_t)v][i], &tmp))
              r = fail(QC_ERR_CUDA, "loopback shard box tensor map");
          }
        }
      }
    }
    if (r != QC_OK) return r;
    P->passes += (int64_t)st.seg->passes.size();
    if (seg_pair >= 0) P->pair_segments++;
    P->steps.push_back(std::move(st));
    seg.clear();
    seg_pair = -1;
    return QC_OK;
  };
  for (size_t i = 0; i < n_ops; ++i) {
    const qc_gate& op = ops[i];
    if (op.op == QC_SWAP && s->relabel) {
      std::swap(lay[op.qubits[0]], lay[op.qubits[1]]);
      std::swap(rel[op.qubits[0]], rel[op.qubits[1]]);
      inv[lay[op.qubits[0]]] = op.qubits[0];
      inv[lay[op.qubits[1]]] = op.qubits[1];
      P->relabels++;
      continue;
    }
    const uint64_t nd = op_nondiag_mask(op, mt);
    if (s->xmode == 2) {
      // pair passes: a gate with exactly one non-diagonal rank-bit qubit runs
      // in a pair segment on that rank bit (no exchange, layout unchanged)
      int gbit = -1, ng = 0;
      for (int q = 0; q < n; ++q)
        if ((nd & (1ull << q)) && lay[q] >= nl) {
          gbit = lay[q];
          ++ng;
        }
      if (ng == 1) {
        if (seg_pair != gbit) {
          if (seg_pair >= 0) {
            qc_status r = flush();
            if (r != QC_OK) return r;
          }
          seg_pair = gbit;  // a pending local segment joins the pair segment
        }
        seg.push_back(lower(op, lay, mt));
        continue;
      }
    }
    uint64_t op_qubits = 0;
    {
      int qs[QC_MGATE_MAX_QUBITS];
      const int nq = qc::op_qubits(op, mt, qs);
      for (int t = 0; t < nq; ++t) op_qubits |= 1ull << qs[t];
    }
    for (int q = 0; q < n; ++q) {
      if (!(nd & (1ull << q)) || lay[q] < nl) continue;
      // qubit q is non-diagonal and global: bring it to local bit L
      const int g = lay[q];
      int victim = -1;
      long best = -1;
      for (int p = 0; p < nl; ++p) {
        const int vq = inv[p];
        if (op_qubits & (1ull << vq)) continue;  // must stay local for this op
        const long nu = next_use(vq, i);
        const long score = nu * 2 + (p == L ? 1 : 0);  // prefer the slot itself on ties
        if (score > best) {
          best = score;
          victim = p;
        }
      }
      if (victim < 0) return fail(QC_ERR_UNSUPPORTED, "no local qubit free for an exchange");
      if (victim != L) {  // physical SWAP of two local bits, fused into the segment
        PGate sw;
        sw.kind = GK::SWAP2;
        sw.t0 = std::max(victim, L);
        sw.t1 = std::min(victim, L);
        seg.push_back(sw);
        const int qa = inv[victim], qb = inv[L];
        std::swap(lay[qa], lay[qb]);
        inv[lay[qa]] = qa;
        inv[lay[qb]] = qb;
      }
      qc_status r = flush();
      if (r != QC_OK) return r;
      DistPlan::Step ex;
      ex.kind = 1;
      ex.g = g;
      ex.l = L;
      P->steps.push_back(std::move(ex));
      P->exchanges++;
      const int qg = inv[g], ql = inv[L];
      std::swap(lay[qg], lay[ql]);
      inv[lay[qg]] = qg;
      inv[lay[ql]] = ql;
    }
    PGate pg = lower(op, lay, mt);
    seg.push_back(pg);
  }
  // Restore: undo the exchanges' permutation so the run ends in the layout
  // the SWAP relabels alone give (so a repeated circuit starts from a layout
  // it has seen: its sharded plan, JIT kernels and timing are reused instead
  // of re-planned every run).  Rank bits first -- the qubit each should hold
  // is brought to the exchange slot L (a local SWAP2 fused into the last
  // segment, or an exchange if it sits on another rank bit) and exchanged
  // into place -- then the local bits by SWAP2s in the last segment.
  auto swap_local = [&](int a, int b) {  // physical SWAP of two local bits
    if (a == b) return;
    PGate sw;
    sw.kind = GK::SWAP2;
    sw.t0 = std::max(a, b);
    sw.t1 = std::min(a, b);
    seg.push_back(sw);
    const int qa = inv[a], qb = inv[b];
    std::swap(lay[qa], lay[qb]);
    inv[lay[qa]] = qa;
    inv[lay[qb]] = qb;
  };
  auto exchange = [&](int g) -> qc_status {  // rank bit g <-> L
    qc_status fr = flush();
    if (fr != QC_OK) return fr;
    DistPlan::Step ex;
    ex.kind = 1;
    ex.g = g;
    ex.l = L;
    ex.restore = true;
    P->steps.push_back(std::move(ex));
    P->exchanges++;
    P->restore_exchanges++;
    const int qg = inv[g], ql = inv[L];
    std::swap(lay[qg], lay[ql]);
    inv[lay[qg]] = qg;
    inv[lay[ql]] = ql;
    return QC_OK;
  };
  static const bool restore = !getenv("QC_DIST_RESTORE") || atoi(getenv("QC_DIST_RESTORE")) != 0;
  int rinv[64];
  for (int q = 0; q < n; ++q) rinv[rel[q]] = q;
  for (int g = nl; g < n && restore; ++g) {
    const int want = rinv[g];
    if (inv[g] == want) continue;
    if (lay[want] >= nl) {  // on a later rank bit: bring it to L first
      qc_status er = exchange(lay[want]);
      if (er != QC_OK) return er;
    } else {
      swap_local(lay[want], L);
    }
    qc_status er = exchange(g);
    if (er != QC_OK) return er;
  }
  for (int p = 0; p < nl && restore; ++p)
    if (inv[p] != rinv[p]) swap_local(p, lay[rinv[p]]);
  qc_status r = flush();
  if (r != QC_OK) return r;
  P->layout_out.assign(lay, lay + n);
  return QC_OK;
}

// A pair segment (kind 2) on rank bit g: every pass is planned over the nl
// local bits + the pair bit (plan bit nl).  The two ranks r, r ^ 2^(g-nl)
// split each pass's tiles by the top tile-index bit (rank with pair bit v
// takes half v).  A pass whose tile holds the pair bit reads and writes both
// shards (its own and, over NVLink, the partner's: the collective is fused
// into the pass -- no staging, no layout change); its tile halves come from
// the two buffers.  Every other pass's half-v tiles lie in rank v's own
// shard.  A pair pass is bracketed by pairwise barriers (the partner's
// previous pass on its shard is done before, and its pair pass is done with
// our shard after).  Loopback: all virtual ranks, pass by pass.
qc_status enqueue_pair_segment(qc_state* s, const DistPlan::Step& st) {
  PlanEntry* e = st.seg.get();
  const int nl = s->n_loc, j = st.g - nl;
  const uint64_t pm = 1ull << nl;
  struct Buf {
    void* ptr;
    uint64_t ab;
    bool peer;
    int vr;  // loopback virtual rank whose shard this is (-1: NCCL rank buffers)
  };
  auto tmap_of = [&](const Buf& b, size_t i) -> const QcTmap& {
    if (b.vr >= 0)  // loopback: the virtual rank's own shard maps
      return e->passes[i].g4 == 2 ? e->vr_box[(size_t)b.vr][i] : e->vr_row[(size_t)b.vr];
    if (b.peer) return e->tmaps_peer.empty() ? e->tmap_peer : e->tmaps_peer[i];
    return e->tmaps.empty() ? e->tmap : e->tmaps[i];
  };
  auto launch_rank = [&](int r, size_t i) -> int {
    const int partner = r ^ (1 << j), v = (r >> j) & 1;
    PassDesc pd = e->passes[i];
    // rank bits in plan space: global bit g's value sits at plan bit nl (it is
    // the pair bit, variable: not a constant) and global bit nl's at g
    uint64_t R = (uint64_t)r << nl;
    if (st.g != nl) {
      const uint64_t bn = (R >> nl) & 1ull, bg = (R >> st.g) & 1ull;
      R = (R & ~(pm | (1ull << st.g))) | (bn << st.g) | (bg << nl);
    }
    pd.rank_bits = R & ~pm;
    const uint64_t half = pd.n_tiles / 2;
    pd.n_tiles = half;
    pd.tile0 = v ? half : 0;
    Buf mine{s->d, 0, false, -1}, peer{nullptr, 0, true, -1};
    if (s->dist == 1) {  // loopback: every shard addressed as its own buffer (as the P2P peers)
      const size_t sb = (size_t)(s->dbl ? 16 : 8) << nl;
      mine = Buf{(char*)s->d + (size_t)r * sb, 0, false, r};
      peer = Buf{(char*)s->d + (size_t)partner * sb, 0, false, partner};
    } else {
      peer.ptr = s->peers[(size_t)partner];
    }
    QcTmapSet tms;
    if (!pd.grp) {
      pd.addr_bits = mine.ab;
      tms.m[0] = tmap_of(mine, i);
      return launch_pass(s, e, i, pd, mine.ptr, tms, s->stream);
    }
    const Buf* hb[2] = {v ? &peer : &mine, v ? &mine : &peer};  // sub-tile h = pair bit h
    for (int h = 0; h < 2; ++h) {
      tms.m[h] = tmap_of(*hb[h], i);
      pd.sub_addr[h] = hb[h]->ab;
      pd.sub_state[h] = (uint64_t)(uintptr_t)hb[h]->ptr;
    }
    return launch_pass(s, e, i, pd, hb[0]->ptr, tms, s->stream);
  };
  const size_t np = e->passes.size();
  if (s->dist == 1) {
    for (size_t i = 0; i < np; ++i)
      for (int r = 0; r < s->world; ++r)
        if (const int rc = launch_rank(r, i)) return cuda_fail(s, rc, "pair segment pass (loopback)");
    return QC_OK;
  }
  const int partner = s->rank ^ (1 << j);
  bool prev_pair = false;
  for (size_t i = 0; i < np; ++i) {
    const bool pr = e->passes[i].grp != 0;
    if (pr && !prev_pair) {
      const qc_status b = pair_barrier(s, partner);
      if (b != QC_OK) return b;
    }
    if (const int rc = launch_rank(s->rank, i)) return cuda_fail(s, rc, "pair segment pass");
    if (pr) {
      const qc_status b = pair_barrier(s, partner);
      if (b != QC_OK) return b;
    }
    prev_pair = pr;
  }
  return QC_OK;
}

// Stream-ordered barrier of all ranks (a 1-byte NCCL all-reduce): every
// rank's earlier work on its shard is done before anyone's later work.
qc_status world_barrier(qc_state* s) {
  const int r = nccl().all_reduce(s->d_token, s->d_token, 1, kNcclUint8, kNcclSum, s->nccl_comm, s->stream);
  return r ? nccl_fail(s, r, "world barrier") : QC_OK;
}

}  // namespace

// Tile split of one group-plan pass for rank r (host arithmetic, also
// qc_debug_group_split).  T: the pass's tile bit set over the n-bit index;
// rank bits are nl..nl+p-1.  G = the rank bits in T (j of them: the tile's
// top j local bits), O = the other rank bits (the top p-j tile-index bits,
// outer positions ascending).  Rank r takes the n_tiles / 2^p tiles whose
// O bits equal r's and whose next j index bits equal r's G bits; sub-tile h
// (G bits = h) of such a tile lives in rank owner[h] (r's O bits, G bits h).
GroupSplit group_split(int nl, int p, uint64_t T, uint64_t n_tiles, int r) {
  auto pext = [](uint32_t x, uint32_t m) {
    uint32_t v = 0;
    for (int b = 0, o = 0; b < 32; ++b)
      if ((m >> b) & 1u) v |= ((x >> b) & 1u) << o++;
    return v;
  };
  auto pdep = [](uint32_t x, uint32_t m) {
    uint32_t v = 0;
    for (int b = 0, o = 0; b < 32; ++b)
      if ((m >> b) & 1u) v |= ((x >> o++) & 1u) << b;
    return v;
  };
  const uint32_t all = (1u << p) - 1u;
  const uint32_t G = (uint32_t)(T >> nl) & all;
  GroupSplit sp;
  sp.j = std::popcount(G);
  const int tb = std::countr_zero(n_tiles);
  sp.count = n_tiles >> p;
  sp.tile0 = ((uint64_t)pext((uint32_t)r, all & ~G) << (tb - (p - sp.j))) |
             ((uint64_t)pext((uint32_t)r, G) << (tb - p));
  for (int h = 0; h < 8; ++h) sp.owner[h] = h < (1 << sp.j) ? (int)(((uint32_t)r & ~G) | pdep((uint32_t)h, G)) : -1;
  return sp;
}

namespace {

// A group plan (kind 3) over all n bits.  Pass i on rank r: the tile's rank
// bits G (|G| = j) are its top j local bits; the other rank bits O are the
// top p-j tile-index bits.  Rank r takes the tiles whose O bits equal its own
// and, of those, the 1/2^j whose next j index bits equal its G bits -- one
// contiguous range of n_tiles / P tiles.  Sub-tile h of such a tile lives in
// the rank with r's O bits and G bits = h; a pass with j = 0 stays in the
// rank's own shard.  Passes with j > 0 are bracketed by world barriers
// (NCCL); the loopback runs all virtual ranks pass by pass.
qc_status enqueue_group_plan(qc_state* s, const DistPlan::Step& st) {
  PlanEntry* e = st.seg.get();
  const int nl = s->n_loc, p = std::countr_zero((unsigned)s->world);
  const size_t shard_bytes = (size_t)(s->dbl ? 16 : 8) << nl;
  auto buf_of = [&](int q) -> void* {
    return s->dist == 1 ? (void*)((char*)s->d + (size_t)q * shard_bytes) : s->peers[(size_t)q];
  };
  auto map_of = [&](int q, size_t i) -> const QcTmap& {
    return e->passes[i].g4 == 2 ? e->vr_box[(size_t)q][i] : e->vr_row[(size_t)q];
  };
  auto launch_rank = [&](int r, size_t i) -> int {
    PassDesc pd = e->passes[i];
    const GroupSplit sp = group_split(nl, p, pass_tile_set(pd), pd.n_tiles, r);
    const int j = sp.j;
    pd.n_tiles = sp.count;
    pd.tile0 = sp.tile0;
    pd.rank_bits = 0;
    pd.addr_bits = 0;
    QcTmapSet tms;
    if (!j) {
      tms.m[0] = map_of(r, i);
      return launch_pass(s, e, i, pd, buf_of(r), tms, s->stream);
    }
    for (int h = 0; h < (1 << j); ++h) {
      tms.m[h] = map_of(sp.owner[h], i);
      pd.sub_addr[h] = 0;
      pd.sub_state[h] = (uint64_t)(uintptr_t)buf_of(sp.owner[h]);
    }
    return launch_pass(s, e, i, pd, buf_of(sp.owner[0]), tms, s->stream);
  };
  const size_t np = e->passes.size();
  if (s->dist == 1) {
    for (size_t i = 0; i < np; ++i)
      for (int r = 0; r < s->world; ++r)
        if (const int rc = launch_rank(r, i)) return cuda_fail(s, rc, "group plan pass (loopback)");
    return QC_OK;
  }
  bool prev = false;
  for (size_t i = 0; i < np; ++i) {
    const bool spans = e->passes[i].grp != 0;
    if (spans && !prev) {
      const qc_status b = world_barrier(s);
      if (b != QC_OK) return b;
    }
    if (const int rc = launch_rank(s->rank, i)) return cuda_fail(s, rc, "group plan pass");
    if (spans) {
      const qc_status b = world_barrier(s);
      if (b != QC_OK) return b;
    }
    prev = spans;
  }
  return QC_OK;
}

qc_status enqueue_dist(qc_state* s, DistPlan* P) {
  const uint64_t nloc_amps = 1ull << s->n_loc;
  for (auto& st : P->steps) {
    if (st.kind == 3) {
      const qc_status r = enqueue_group_plan(s, st);
      if (r != QC_OK) return r;
      continue;
    }
    if (st.kind == 2) {
      const qc_status r = enqueue_pair_segment(s, st);
      if (r != QC_OK) return r;
      continue;
    }
    if (st.kind == 1) {
      const qc_status r = dist_exchange(s, st.g, st.l);
      if (r != QC_OK) return r;
      continue;
    }
    if (s->dist == 1) {
      for (int v = 0; v < s->world; ++v) {
        const uint64_t rb = (uint64_t)v * nloc_amps;
        const int e = enqueue_entry(s, st.seg.get(), s->stream, s->d, rb, rb);
        if (e) return cuda_fail(s, e, "fused pass (loopback shard)");
      }
    } else {
      const uint64_t rb = (uint64_t)s->rank * nloc_amps;
      const int e = enqueue_entry(s, st.seg.get(), s->stream, s->d, rb, 0);
      if (e) return cuda_fail(s, e, "fused pass (shard)");
    }
  }
  return QC_OK;
}

}  // namespace

// Host-only schedule for tests (qc_debug.h): steps as (kind, g, l, gates).
qc_status dist_schedule_dry(int n, int world, int relabel, const qc_gate* ops, size_t n_ops,
                            std::vector<int>& out, std::vector<int>& layout_out, const MTable* mt, int xmode) {
  qc_state s;
  s.n = n;
  s.world = world;
  s.n_loc = n - std::countr_zero((unsigned)world);
  s.relabel = relabel;
  s.xmode = xmode;
  s.dist = 1;
  for (int q = 0; q < n; ++q) s.layout[q] = n - 1 - q;
  DistPlan P;
  const qc_status r = build_dist_plan(&s, ops, n_ops, &P, mt, true);
  if (r != QC_OK) return r;
  for (auto& st : P.steps) {
    out.push_back(st.kind);
    out.push_back(st.g);
    out.push_back(st.l);
    out.push_back(st.kind != 1 ? (int)st.seg->fused_gates : (st.restore ? 1 : 0));
  }
  layout_out = P.layout_out;
  return QC_OK;
}

qc_status run_dist(qc_state* s, const qc_gate* ops, size_t n_ops, const MTable* mt) {
  {
    const qc_status c = ensure_fused_configured(s);
    if (c != QC_OK) return c;
  }
  const uint64_t salt = 0xd157ull ^ ((uint64_t)s->relabel << 2) ^ ((uint64_t)s->block_fusion << 3) ^
                        ((uint64_t)s->tile_bits << 8) ^ ((uint64_t)s->row_bits << 16) ^
                        ((uint64_t)s->tma_mode << 24) ^ ((uint64_t)s->jit << 28) ^ ((uint64_t)s->remap << 32) ^
                        ((uint64_t)s->ctas << 36) ^ ((uint64_t)s->xmode << 44) ^ ((uint64_t)s->fusion << 56);
  std::vector<uint8_t> mkey = mtable_key(ops, n_ops, mt);
  uint64_t key = hash_ops(ops, n_ops, s->layout, s->n, salt);
  for (uint8_t b : mkey) key = (key ^ b) * 0x100000001b3ull;
  DistPlan* P = nullptr;
  if (!s->dcache) s->dcache = new DistCache();
  auto& dplans = s->dcache->plans;
  auto it = dplans.find(key);
  if (it != dplans.end() && it->second->ops.size() == n_ops &&
      std::memcmp(it->second->ops.data(), ops, n_ops * sizeof(qc_gate)) == 0 && it->second->mkey == mkey &&
      std::memcmp(it->second->layout_in.data(), s->layout, sizeof(int) * s->n) == 0) {
    P = it->second.get();
  } else {
    auto np = std::make_unique<DistPlan>();
    np->ops.assign(ops, ops + n_ops);
    np->mkey = std::move(mkey);
    np->layout_in.assign(s->layout, s->layout + s->n);
    const qc_status r = build_dist_plan(s, ops, n_ops, np.get(), mt);
    if (r != QC_OK) return r;
    P = np.get();
    if (dplans.size() > 32) dplans.clear();
    dplans[key] = std::move(np);
  }
  P->uses++;
  for (auto& st : P->steps) {
    if (st.kind == 1) continue;
    st.seg->uses = P->uses;
    const qc_status r = maybe_jit(s, st.seg.get());
    if (r != QC_OK) return r;
  }
  const qc_status r = enqueue_dist(s, P);
  if (r != QC_OK) return r;
  std::memcpy(s->layout, P->layout_out.data(), sizeof(int) * s->n);
  int64_t launches = 0;
  bool jit = true;
  for (auto& st : P->steps)
    if (st.kind != 1) {
      launches += (int64_t)st.seg->passes.size() * (s->dist == 1 ? s->world : 1);
      jit = jit && st.seg->jit_state == 1;
    }
  s->last_passes = P->passes;
  s->last_launches = launches;
  s->last_relabels = P->relabels;
  s->last_exchanges = P->exchanges;
  s->last_pair_segments = P->pair_segments;
  s->last_graph = 0;
  s->last_jit = jit ? 1 : 0;
  return QC_OK;
}

// Restore the canonical layout (collective): local pairs by SWAP2 kernels on
// each shard, pairs involving rank bits by exchanges through local bit n_loc-1.
qc_status dist_canonicalize(qc_state* s) {
  const int n = s->n, nl = s->n_loc, L = nl - 1;
  auto phys_swap = [&](int a, int b) -> qc_status {  // swap physical bits a, b (a != b)
    if (a < nl && b < nl) {
      PGate g;
      g.kind = GK::SWAP2;
      g.t0 = a;
      g.t1 = b;
      if (s->dist == 1) {
        // loopback: the buffer is the whole state, a local bit swap is a swap on n bits
        const int e = launch_gate(s->d, n, s->dbl, g, s->stream);
        if (e) return cuda_fail(s, e, "canonicalize swap");
      } else {
        const int e = launch_gate(s->d, nl, s->dbl, g, s->stream);
        if (e) return cuda_fail(s, e, "canonicalize swap");
      }
      return QC_OK;
    }
    if (a >= nl && b >= nl) {  // two rank bits: through the slot
      qc_status r = dist_exchange(s, a, L);
      if (r == QC_OK) r = dist_exchange(s, b, L);
      if (r == QC_OK) r = dist_exchange(s, a, L);
      return r;
    }
    const int g = a >= nl ? a : b, l = a >= nl ? b : a;
    if (l == L) return dist_exchange(s, g, L);
    // g <-> l == (l<->L) (g<->L) (l<->L)
    qc_status r = QC_OK;
    PGate sw;
    sw.kind = GK::SWAP2;
    sw.t0 = L;
    sw.t1 = l;
    auto local_sw = [&]() -> qc_status {
      const int e = launch_gate(s->d, s->dist == 1 ? n : nl, s->dbl, sw, s->stream);
      return e ? cuda_fail(s, e, "canonicalize swap") : QC_OK;
    };
    r = local_sw();
    if (r == QC_OK) r = dist_exchange(s, g, L);
    if (r == QC_OK) r = local_sw();
    return r;
  };
  for (int q = 0; q < n; ++q) {
    const int want = n - 1 - q;
    if (s->layout[q] == want) continue;
    int q2 = -1;
    for (int u = 0; u < n; ++u)
      if (s->layout[u] == want) q2 = u;
    const qc_status r = phys_swap(s->layout[q], want);
    if (r != QC_OK) return r;
    s->layout[q2] = s->layout[q];
    s->layout[q] = want;
  }
  return QC_OK;
}

}  // namespace qc
