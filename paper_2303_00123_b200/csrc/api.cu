// api.cu -- the C ABI of include/qc.h: validation, lowering, planning,
// launching, I/O.  Host code only (kernels live in kernels_*.cu).
#include <cuda_runtime.h>

#include <bit>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "qc_internal.h"
#include "state.h"
#include "../../include/qc_debug.h"

using namespace qc;

namespace qc {

thread_local std::string g_err;

qc_status fail(qc_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

const int kArity[16] = {1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 1, 2, 2, 3};
const int kNctrl[16] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 0, 0, 1, 0, 2};
const char* kName[16] = {"H", "X", "Y", "Z", "P", "RX", "RY", "RZ",
                         "CNOT", "CZ", "CP", "SWAP", "U1", "CU1", "U2", "CCX"};

constexpr int kMaxDevices = 64;

size_t amp_bytes(const qc_state* s) { return s->dbl ? 16 : 8; }

void canonical_layout(qc_state* s) {
  for (int q = 0; q < s->n; ++q) s->layout[q] = s->n - 1 - q;
}
bool layout_is_canonical(const qc_state* s) {
  for (int q = 0; q < s->n; ++q)
    if (s->layout[q] != s->n - 1 - q) return false;
  return true;
}

qc_status check_state(qc_state* s) {
  if (!s) return fail(QC_ERR_INVALID_ARG, "state is NULL");
  if (s->failed) return fail(QC_ERR_STATE_FAILED, "state failed earlier (asynchronous CUDA error)");
  cudaError_t e = cudaSetDevice(s->device);
  if (e != cudaSuccess) return fail(QC_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  return QC_OK;
}

qc_status cuda_fail(qc_state* s, int e, const char* what) {
  if (s) s->failed = true;
  return fail(QC_ERR_CUDA, "%s: %s", what, cudaGetErrorString((cudaError_t)e));
}

// A generic gate (qc_mgate) -> validated copy.
qc_status copy_mgate(int n, const qc_mgate& g, size_t idx, MGate* out) {
  if (g.flags != 0) return fail(QC_ERR_INVALID_ARG, "mgate %zu: flags must be 0", idx);
  if (g.n_targ < 1 || g.n_targ > QC_MGATE_MAX_TARGETS)
    return fail(QC_ERR_INVALID_ARG, "mgate %zu: n_targ=%d outside [1,%d]", idx, g.n_targ, QC_MGATE_MAX_TARGETS);
  if (g.n_ctrl < 0 || g.n_ctrl + g.n_targ > QC_MGATE_MAX_QUBITS)
    return fail(QC_ERR_INVALID_ARG, "mgate %zu: n_ctrl=%d (n_ctrl + n_targ <= %d)", idx, g.n_ctrl,
                QC_MGATE_MAX_QUBITS);
  const int nq = g.n_ctrl + g.n_targ;
  for (int t = 0; t < nq; ++t) {
    if (g.qubits[t] < 0 || g.qubits[t] >= n)
      return fail(QC_ERR_INVALID_ARG, "mgate %zu: qubit %d out of range [0,%d)", idx, g.qubits[t], n);
    for (int u = 0; u < t; ++u)
      if (g.qubits[u] == g.qubits[t]) return fail(QC_ERR_INVALID_ARG, "mgate %zu: qubit %d repeated", idx, g.qubits[t]);
  }
  if (!g.matrix) return fail(QC_ERR_INVALID_ARG, "mgate %zu: matrix is NULL", idx);
  const int d = 1 << g.n_targ;
  out->n_ctrl = g.n_ctrl;
  out->n_targ = g.n_targ;
  std::memset(out->qubits, 0, sizeof out->qubits);
  for (int t = 0; t < nq; ++t) out->qubits[t] = g.qubits[t];
  out->ctrl_state = g.n_ctrl >= 32 ? g.ctrl_state : (g.ctrl_state & ((1u << g.n_ctrl) - 1u));
  out->m.resize((size_t)d * d);
  for (int e = 0; e < d * d; ++e) {
    if (!std::isfinite(g.matrix[2 * e]) || !std::isfinite(g.matrix[2 * e + 1]))
      return fail(QC_ERR_INVALID_ARG, "mgate %zu: matrix entry %d not finite", idx, e);
    out->m[e] = cd(g.matrix[2 * e], g.matrix[2 * e + 1]);
  }
  return QC_OK;
}

std::vector<uint8_t> mtable_key(const qc_gate* ops, size_t n_ops, const MTable* mt) {
  std::vector<uint8_t> k;
  if (!mt) return k;
  auto put = [&](const void* p, size_t b) {
    const uint8_t* c = reinterpret_cast<const uint8_t*>(p);
    k.insert(k.end(), c, c + b);
  };
  for (size_t i = 0; i < n_ops; ++i) {
    if (ops[i].op != QC_MGATE) continue;
    const MGate& g = (*mt)[(size_t)ops[i].qubits[0]];
    put(&g.n_ctrl, sizeof g.n_ctrl);
    put(&g.n_targ, sizeof g.n_targ);
    put(g.qubits, sizeof(int) * (size_t)(g.n_ctrl + g.n_targ));
    put(&g.ctrl_state, sizeof g.ctrl_state);
    put(g.m.data(), sizeof(cd) * g.m.size());
  }
  return k;
}

int op_qubits(const qc_gate& g, const MTable* mt, int* out) {
  if (g.op == QC_MGATE) {
    const MGate& m = (*mt)[(size_t)g.qubits[0]];
    for (int t = 0; t < m.n_ctrl + m.n_targ; ++t) out[t] = m.qubits[t];
    return m.n_ctrl + m.n_targ;
  }
  for (int t = 0; t < kArity[g.op]; ++t) out[t] = g.qubits[t];
  return kArity[g.op];
}

// Logical non-diagonal targets (a diagonal gate never needs its qubit local).
uint64_t op_nondiag_mask(const qc_gate& g, const MTable* mt) {
  switch (g.op) {
    case QC_Z: case QC_P: case QC_RZ: case QC_CZ: case QC_CP: return 0;
    case QC_SWAP: case QC_U2: return (1ull << g.qubits[0]) | (1ull << g.qubits[1]);
    case QC_MGATE: {
      const MGate& m = (*mt)[(size_t)g.qubits[0]];
      if (m.n_targ == 1 && m.m[1] == cd(0) && m.m[2] == cd(0)) return 0;
      uint64_t r = 0;
      for (int t = m.n_ctrl; t < m.n_ctrl + m.n_targ; ++t) r |= 1ull << m.qubits[t];
      return r;
    }
    default: return 1ull << g.qubits[kNctrl[g.op]];
  }
}

qc_status validate_gate(int n, const qc_gate& g, size_t idx, const MTable* mt) {
  if (g.op == QC_MGATE) {
    if (g.flags != 0) return fail(QC_ERR_INVALID_ARG, "op %zu: flags must be 0", idx);
    if (!mt || g.qubits[0] < 0 || (size_t)g.qubits[0] >= mt->size())
      return fail(QC_ERR_INVALID_ARG, "op %zu (MGATE): index %d outside the mgate table (%zu)", idx, g.qubits[0],
                  mt ? mt->size() : (size_t)0);
    return QC_OK;
  }
  if (g.op < 0 || g.op > 15) return fail(QC_ERR_INVALID_ARG, "op %zu: unknown op code %d", idx, g.op);
  if (g.flags != 0) return fail(QC_ERR_INVALID_ARG, "op %zu: flags must be 0", idx);
  const int k = kArity[g.op];
  for (int t = 0; t < k; ++t) {
    if (g.qubits[t] < 0 || g.qubits[t] >= n)
      return fail(QC_ERR_INVALID_ARG, "op %zu (%s): qubit %d out of range [0,%d)", idx, kName[g.op],
                  g.qubits[t], n);
    for (int u = 0; u < t; ++u)
      if (g.qubits[u] == g.qubits[t])
        return fail(QC_ERR_INVALID_ARG, "op %zu (%s): qubit %d repeated", idx, kName[g.op], g.qubits[t]);
  }
  const bool has_theta = g.op == QC_P || g.op == QC_RX || g.op == QC_RY || g.op == QC_RZ || g.op == QC_CP;
  if (has_theta && !std::isfinite(g.theta))
    return fail(QC_ERR_INVALID_ARG, "op %zu (%s): theta is not finite", idx, kName[g.op]);
  const int nm = g.op == QC_U2 ? 32 : ((g.op == QC_U1 || g.op == QC_CU1) ? 8 : 0);
  for (int i = 0; i < nm; ++i)
    if (!std::isfinite(g.m[i]))
      return fail(QC_ERR_INVALID_ARG, "op %zu (%s): matrix entry %d not finite", idx, kName[g.op], i);
  return QC_OK;
}

// Generic gate -> physical-bit kernel class; the exact structure of a 2x2
// target matrix picks the class (diagonal -> phase, X pattern -> move).
PGate lower_mgate(const MGate& g, const int* layout) {
  PGate p;
  for (int t = 0; t < g.n_ctrl; ++t) {
    const int b = layout[g.qubits[t]];
    p.cmask |= 1ull << b;
    if ((g.ctrl_state >> t) & 1u) p.cval |= 1ull << b;
  }
  const int* tq = g.qubits + g.n_ctrl;
  const cd* M = g.m.data();
  auto zero = [](cd z) { return z.real() == 0.0 && z.imag() == 0.0; };
  auto one = [](cd z) { return z.real() == 1.0 && z.imag() == 0.0; };
  if (g.n_targ == 1) {
    p.t0 = layout[tq[0]];
    if (zero(M[1]) && zero(M[2])) {
      p.kind = GK::DIAG1;
      p.m[0] = M[0];
      p.m[1] = M[3];
      p.d0_is_one = one(M[0]);
    } else if (zero(M[0]) && zero(M[3]) && one(M[1]) && one(M[2])) {
      p.kind = GK::PERM1;
    } else {
      p.kind = GK::DENSE1;
      for (int i = 0; i < 4; ++i) p.m[i] = M[i];
    }
  } else if (g.n_targ == 2) {
    p.kind = GK::DENSE2;
    p.t0 = layout[tq[0]];
    p.t1 = layout[tq[1]];
    for (int i = 0; i < 16; ++i) p.m[i] = M[i];
  } else {
    p.kind = GK::DENSEK;
    p.nt = g.n_targ;
    for (int j = 0; j < g.n_targ; ++j) p.tk[j] = layout[tq[j]];
    p.t0 = p.tk[0];
    p.mk = std::make_shared<const std::vector<cd>>(g.m);
  }
  return p;
}

// Lower one validated gate to a physical-bit kernel class (DESIGN R4 matrices).
PGate lower(const qc_gate& g, const int* layout, const MTable* mt) {
  if (g.op == QC_MGATE) return lower_mgate((*mt)[(size_t)g.qubits[0]], layout);
  PGate p;
  const int nc = kNctrl[g.op];
  for (int t = 0; t < nc; ++t) {
    const int b = layout[g.qubits[t]];
    p.cmask |= 1ull << b;
    if ((g.ctrl_state >> t) & 1u) p.cval |= 1ull << b;
  }
  const int tq = g.qubits[nc];
  p.t0 = layout[tq];
  const double th = g.theta;
  const double c = std::cos(th / 2), s = std::sin(th / 2);
  const double h = 1.0 / std::sqrt(2.0);
  const cd I(0, 1);
  auto dense = [&](cd a, cd b, cd cc, cd d) {
    p.kind = GK::DENSE1;
    p.m[0] = a; p.m[1] = b; p.m[2] = cc; p.m[3] = d;
  };
  auto diag = [&](cd d0, cd d1, bool one) {
    p.kind = GK::DIAG1;
    p.m[0] = d0; p.m[1] = d1;
    p.d0_is_one = one;
  };
  switch (g.op) {
    case QC_H: dense(h, h, h, -h); break;
    case QC_X: case QC_CNOT: case QC_CCX: p.kind = GK::PERM1; break;
    case QC_Y: dense(0, -I, I, 0); break;
    case QC_Z: case QC_CZ: diag(1.0, -1.0, true); break;
    case QC_P: case QC_CP: diag(1.0, std::exp(I * th), true); break;
    case QC_RX: dense(c, -I * s, -I * s, c); break;
    case QC_RY: dense(c, -s, s, c); break;
    case QC_RZ: diag(std::exp(-I * (th / 2)), std::exp(I * (th / 2)), false); break;
    case QC_U1: case QC_CU1:
      dense(cd(g.m[0], g.m[1]), cd(g.m[2], g.m[3]), cd(g.m[4], g.m[5]), cd(g.m[6], g.m[7]));
      break;
    case QC_SWAP:
      p.kind = GK::SWAP2;
      p.t0 = layout[g.qubits[0]];
      p.t1 = layout[g.qubits[1]];
      break;
    case QC_U2:
      p.kind = GK::DENSE2;
      p.t0 = layout[g.qubits[0]];
      p.t1 = layout[g.qubits[1]];
      for (int i = 0; i < 16; ++i) p.m[i] = cd(g.m[2 * i], g.m[2 * i + 1]);
      break;
  }
  return p;
}

uint64_t hash_ops(const qc_gate* ops, size_t n, const int* layout, int nq, uint64_t salt) {
  uint64_t h = 0xcbf29ce484222325ull ^ salt;
  auto mix = [&](uint64_t w) {
    h ^= w;
    h *= 0x100000001b3ull;
    h ^= h >> 29;
  };
  const uint64_t* w = reinterpret_cast<const uint64_t*>(ops);
  const size_t nw = n * sizeof(qc_gate) / 8;
  for (size_t i = 0; i < nw; ++i) mix(w[i]);
  for (int q = 0; q < nq; ++q) mix((uint64_t)layout[q] + 977ull * q);
  mix(n);
  return h;
}

// Per-pass FP64 budget of the planner (flops per amplitude, plan_fused).
double pass_flops_budget(bool dbl) {
  const char* e = getenv("QC_PASS_FLOPS");
  if (e) return atof(e);
  (void)dbl;
  return 0;
}

void plan_geometry(const qc_state* s, int n_plan, int* k_out, int* rb_out, int* ctas_out) {
  int k = s->tile_bits ? s->tile_bits : (s->dbl ? 12 : 13);
  if (s->dbl && k > 12) k = 12;  // two 2^k tiles (one per compute group) must fit in smem
  if (k > n_plan) k = n_plan;
  int rb = s->row_bits ? s->row_bits : (s->dbl ? 6 : 7);  // 1 KiB rows: half the TMA requests of 512 B rows
  if (rb > k - 2) rb = k - 2;
  if (rb < 1) rb = 1;
  *k_out = k;
  *rb_out = rb;
  *ctas_out = s->ctas ? s->ctas : sm_count();
}

// Tile bit set of a planned pass: the row bits plus its hi bits.
uint64_t pass_tile_set(const PassDesc& d) {
  uint64_t T = (1ull << d.rb) - 1;
  for (int j = 0; j < d.n_hi; ++j) T |= 1ull << d.hi_pos[j];
  return T;
}

// Host cost model of a plan (seconds per amplitude-normalised unit): per pass
// sqrt(H^2 + F^2), H = 2 Ns / the transport's rate, F = its fused flops / the
// ALU rate.  Rates from round-2 B200 measurements: TMA box
// transport 4.1 / 4.55 / 5.3 / 5.7 TB/s when the tile's innermost run is 64 /
// 128 / 256 / >= 512 B; gather4 rows 5.6 (1 KiB), 4.6 (512 B), 3.5 (less);
// fused passes ~34 (c128) / ~52 (c64) algorithmic TFLOP/s (after the full register frames).
double plan_cost_model(const FusedPlan& fp, int n, bool dbl, bool box) {
  const double ab = dbl ? 16 : 8, N = std::ldexp(1.0, n);
  double t = 0;
  for (const FusedPassPlan& pp : fp.passes) {
    const PassDesc& d = pp.desc;
    const uint64_t T = pass_tile_set(d);
    PassDesc tmp = d;
    double bw;
    if (box && make_box_tmap(nullptr, n, dbl, T, nullptr, &tmp)) {
      const int run0 = std::countr_one(T);
      const double inner = ab * std::ldexp(1.0, std::min(run0, dbl ? 7 : 8));
      bw = inner <= 64 ? 4.1e12 : inner <= 128 ? 4.55e12 : (inner <= 256 ? 5.3e12 : 5.7e12);
    } else {
      const double row = ab * std::ldexp(1.0, d.rb);
      bw = row >= 1024 ? 5.6e12 : (row >= 512 ? 4.6e12 : 3.5e12);
    }
    const double H = 2 * ab * N / bw, F = pass_flops_per_amp(pp) * N / (dbl ? 34e12 : 52e12);
    t += std::sqrt(H * H + F * F);
  }
  return t;
}

// Plan the blocks; with row_bits 0 in the box transport, try several row
// widths (narrow rows leave more free tile bits per pass -> fewer passes,
// but slower rows) and keep the plan the cost model prefers -- the widest
// rows within 2 % of the cheapest (the model is only that accurate).
FusedPlan plan_best(int n_plan, int k, int rb_default, int row_bits_opt, bool box, bool dbl,
                    const std::vector<PGate>& blocks, bool remap, int* rb_out) {
  std::vector<int> cands;
  if (row_bits_opt || !box || n_plan <= k) cands.push_back(rb_default);
  else cands = dbl ? std::vector<int>{3, 4, 5, 6} : std::vector<int>{3, 4, 5, 6, 7};
  int need_max = 0;  // a tile holds the row bits plus every non-diagonal target of a gate
  for (const PGate& g : blocks) need_max = std::max(need_max, g.kind == GK::DIAG1 ? 0 : std::popcount(pgate_targets(g)));
  FusedPlan best;
  double best_cost = 1e300;
  int best_rb = -1;
  for (int rb : cands) {
    if (rb > k - 2) rb = k - 2;
    if (rb + need_max > k) rb = k - need_max;
    if (rb < 1) rb = 1;
    if (rb == best_rb) continue;
    FusedPlan fp = plan_fused(n_plan, k, rb, blocks, remap, pass_flops_budget(dbl));
    if (!fp.ok) continue;
    const double c = plan_cost_model(fp, n_plan, dbl, box);
    if (getenv("QC_PLAN_DEBUG"))
      fprintf(stderr, "plan_best: rb %d -> %zu passes, model %.1f ms\n", rb, fp.passes.size(), c * 1e3);
    if (c < best_cost * (best_rb < 0 ? 1.0 : 1.02)) {  // candidates ascend: wider wins near-ties
      best_cost = std::min(c, best_cost);
      best_rb = rb;
      best = std::move(fp);
    }
  }
  if (best_rb < 0) best.ok = false;
  *rb_out = best_rb;
  return best;
}

// Fuse + plan + pack + upload lowered gates over n_plan local bits (bits at or
// above n_plan -- the rank bits of a sharded state -- may appear only as
// controls / diagonal bits).  `tmap_base` / `tmap_bits`: the buffer and index
// width the row tensor map spans.
qc_status build_fused_entry(qc_state* s, const std::vector<PGate>& gates, int n_plan, uint64_t local_mask,
                            PlanEntry* e, void* tmap_base, int tmap_bits, bool remap, uint64_t group_mask,
                            void* peer_base) {
  int k, rb, ctas;
  // plans spanning shards (group_mask = the plan's rank bits): the 2^j ranks
  // split every pass's tiles, so a pass needs >= 2^j tiles (k <= n_plan - j)
  plan_geometry(s, n_plan - std::popcount(group_mask), &k, &rb, &ctas);
  e->ctas = ctas;
  e->tile_bits = k;
  std::vector<PGate> blocks = s->block_fusion ? fuse_blocks(gates, local_mask) : gates;
  e->fused_gates = (int64_t)blocks.size();
  if (blocks.empty()) return QC_OK;
  const bool box = s->tma_mode == 0;
  FusedPlan fp = plan_best(n_plan, k, rb, s->row_bits, box, s->dbl, blocks, remap, &rb);
  if (!fp.ok) return fail(QC_ERR_UNSUPPORTED, "planner failed (k=%d rb=%d)", k, rb);
  e->perm = fp.perm;
  e->flops_per_amp = plan_flops_per_amp(fp);
  void* tb = tmap_base ? tmap_base : s->d;
  const int tbits = tmap_bits ? tmap_bits : n_plan;
  const bool g4 = (s->tma_mode == 0 || s->tma_mode == 2) && make_row_tmap(tb, tbits, rb, s->dbl, &e->tmap) &&
                  (!peer_base || make_row_tmap(peer_base, tbits, rb, s->dbl, &e->tmap_peer));
  e->group_mask = group_mask;
  for (auto& p : fp.passes) {
    p.desc.g4 = g4 ? 1 : 0;
    p.desc.pshift = g4 ? 31 : rb;  // TMA tensor smem dst must be 128-B aligned: no padding
    // rank bits never reach an address (they select the buffer); a pass
    // whose tile holds j of them moves its 2^j sub-tiles separately
    p.desc.addr_strip = group_mask;
    p.desc.grp = std::popcount(pass_tile_set(p.desc) & group_mask);
  }
  if (box) {
    // one TMA box per tile (per sub-tile of a tile spanning shards) where the tile's bit
    // runs fit a 5-D tensor map (else that pass keeps the gather4 rows, or
    // per-row copies)
    e->tmaps.assign(fp.passes.size(), e->tmap);
    if (peer_base) e->tmaps_peer.assign(fp.passes.size(), e->tmap_peer);
    for (size_t i = 0; i < fp.passes.size(); ++i) {
      PassDesc& d = fp.passes[i].desc;
      PassDesc d2 = d;
      const uint64_t T = pass_tile_set(d) & ~group_mask;
      if (make_box_tmap(tb, tbits, s->dbl, T, &e->tmaps[i], &d2) &&
          (!peer_base || make_box_tmap(peer_base, tbits, s->dbl, T, &e->tmaps_peer[i], &d2))) {
        d = d2;
        d.g4 = 2;
        d.pshift = 31;
      }
    }
  }
  for (auto& p : fp.passes)  // a gather4 request (4 rows) must not straddle two sub-tiles
    if (p.desc.grp && p.desc.g4 == 1 && p.desc.k - p.desc.rb - p.desc.grp < 2) {
      p.desc.g4 = 0;
      p.desc.pshift = p.desc.rb;
    }
  std::vector<uint8_t> blob = pack_plan(fp, s->dbl);
  for (auto& p : fp.passes) e->passes.push_back(p.desc);
  e->dbl = s->dbl;
  e->ir = std::make_shared<FusedPlan>(std::move(fp));
  cudaError_t ce = cudaMalloc(&e->d_blob, blob.size());
  if (ce != cudaSuccess) return fail(QC_ERR_OUT_OF_MEMORY, "plan upload: %s", cudaGetErrorString(ce));
  ce = cudaMemcpy(e->d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) return cuda_fail(s, ce, "plan upload");
  return QC_OK;
}

// Build (or fetch) the fused plan for this op list and the current layout.
qc_status get_plan(qc_state* s, const qc_gate* ops, size_t n_ops, const MTable* mt, PlanEntry** out) {
  const int n = s->n;
  int k, rb, ctas;
  plan_geometry(s, n, &k, &rb, &ctas);
  const uint64_t salt = ((uint64_t)s->fusion << 1) ^ ((uint64_t)s->relabel << 2) ^
                        ((uint64_t)s->block_fusion << 3) ^ ((uint64_t)s->jit << 4) ^ ((uint64_t)s->row_bits << 40) ^ ((uint64_t)s->tma_mode << 48) ^ ((uint64_t)s->remap << 52) ^
                        ((uint64_t)k << 8) ^ ((uint64_t)s->dbl << 16) ^ ((uint64_t)ctas << 20);
  std::vector<uint8_t> mkey = mtable_key(ops, n_ops, mt);
  uint64_t key = hash_ops(ops, n_ops, s->layout, n, salt);
  for (uint8_t b : mkey) key = (key ^ b) * 0x100000001b3ull;
  auto it = s->plans.find(key);
  if (it != s->plans.end()) {
    PlanEntry* e = it->second.get();
    if (e->ops.size() == n_ops && std::memcmp(e->ops.data(), ops, n_ops * sizeof(qc_gate)) == 0 &&
        e->mkey == mkey && std::memcmp(e->layout_in.data(), s->layout, n * sizeof(int)) == 0) {
      *out = e;
      return QC_OK;
    }
  }
  auto e = std::make_unique<PlanEntry>();
  e->ops.assign(ops, ops + n_ops);
  e->mkey = std::move(mkey);
  e->layout_in.assign(s->layout, s->layout + n);
  // lower in order, applying SWAP relabels to a running layout
  int lay[64];
  std::memcpy(lay, s->layout, sizeof(int) * n);
  std::vector<PGate> gates;
  gates.reserve(n_ops);
  for (size_t i = 0; i < n_ops; ++i) {
    if (ops[i].op == QC_SWAP && s->relabel) {
      std::swap(lay[ops[i].qubits[0]], lay[ops[i].qubits[1]]);
      e->relabels++;
      continue;
    }
    PGate g = lower(ops[i], lay, mt);
    g.src_op = (int)i;
    gates.push_back(g);
  }
  if (!gates.empty()) {
    const qc_status bs = build_fused_entry(s, gates, n, ~0ull, e.get(), nullptr, 0, s->remap != 0);
    if (bs != QC_OK) return bs;
    if (!e->perm.empty())  // remap swaps moved physical bits: the layout follows the data
      for (int q = 0; q < n; ++q) lay[q] = e->perm[lay[q]];
  }
  e->layout_out.assign(lay, lay + n);
  PlanEntry* raw = e.get();
  if (s->plans.size() > 64) s->plans.clear();
  s->plans[key] = std::move(e);
  *out = raw;
  return QC_OK;
}

int launch_pass(qc_state* s, PlanEntry* e, size_t i, const PassDesc& pd, void* base, const QcTmapSet& tms,
                cudaStream_t st) {
  return (e->jit_state == 1) ? jit_launch(e->jit[i], base, pd, tms, e->ctas, st)
                             : launch_fused_pass(base, s->dbl, pd, e->d_blob, tms, e->ctas, st);
}

// Launch every pass of a fused entry; rank_bits / addr_bits: see PassDesc.
int enqueue_entry(qc_state* s, PlanEntry* e, cudaStream_t st, void* base, uint64_t rank_bits,
                  uint64_t addr_bits) {
  for (size_t i = 0; i < e->passes.size(); ++i) {
    PassDesc pd = e->passes[i];
    pd.rank_bits = rank_bits;
    pd.addr_bits = addr_bits;
    QcTmapSet tms;
    tms.m[0] = e->tmaps.empty() ? e->tmap : e->tmaps[i];
    const int r = launch_pass(s, e, i, pd, base, tms, st);
    if (r) return r;
  }
  return 0;
}

int enqueue_plan(qc_state* s, PlanEntry* e, cudaStream_t st) { return enqueue_entry(s, e, st, s->d, 0, 0); }

// NVRTC-specialise an entry according to the JIT policy: 2nd use by default,
// 1st use when a pass spans >= 2^30 amplitudes -- there the interpreting AOT
// kernel costs more per pass (~25 ms per 2^29 amplitudes over the JIT kernel,
// measured) than compiling every pass on host threads (~1-3 s once per
// process; cubins are cached on disk across processes).
qc_status maybe_jit(qc_state* s, PlanEntry* e) {
  const bool big = !e->passes.empty() && (e->passes[0].n_tiles << e->passes[0].k) >= (1ull << 30);
  if (e->jit_state == 0 && e->ir && (s->jit == 2 || (s->jit == 1 && (e->uses >= 2 || big)))) {
    std::string err;
    if (jit_build(*e->ir, s->dbl, e->jit, err)) {
      e->jit_state = 1;
    } else {
      e->jit_state = -1;
      s->jit_error = err;
      if (s->jit == 2) return fail(QC_ERR_UNSUPPORTED, "JIT specialisation failed: %s", err.c_str());
    }
  }
  return QC_OK;
}

qc_status ensure_fused_configured(qc_state* s) {
  // cudaFuncSetAttribute applies to the current device only: one flag per
  // (device, precision)
  static std::mutex mu;
  static bool configured[kMaxDevices][2] = {};
  if (s->device < 0 || s->device >= kMaxDevices) return fail(QC_ERR_UNSUPPORTED, "device ordinal %d", s->device);
  std::lock_guard<std::mutex> lk(mu);
  if (!configured[s->device][s->dbl]) {
    const int r = fused_configure(s->dbl);
    if (r) return cuda_fail(s, r, "cudaFuncSetAttribute(fused)");
    configured[s->device][s->dbl] = true;
  }
  return QC_OK;
}

qc_status run_fused(qc_state* s, const qc_gate* ops, size_t n_ops, const MTable* mt) {
  {
    const qc_status c = ensure_fused_configured(s);
    if (c != QC_OK) return c;
  }
  PlanEntry* e = nullptr;
  qc_status st = get_plan(s, ops, n_ops, mt, &e);
  if (st != QC_OK) return st;
  e->uses++;
  s->last_graph = 0;
  st = maybe_jit(s, e);
  if (st != QC_OK) return st;
  int r = 0;
  if (s->use_graph && e->uses >= 2 && !e->passes.empty()) {
    if (!e->exec) {
      if (!s->cap_stream) {
        r = cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking);
        if (r) return cuda_fail(s, r, "cudaStreamCreate");
      }
      r = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
      if (r) return cuda_fail(s, r, "cudaStreamBeginCapture");
      const int rl = enqueue_plan(s, e, s->cap_stream);
      r = cudaStreamEndCapture(s->cap_stream, &e->graph);
      if (rl) return cuda_fail(s, rl, "fused launch (capture)");
      if (r) return cuda_fail(s, r, "cudaStreamEndCapture");
      r = cudaGraphInstantiate(&e->exec, e->graph, 0);
      if (r) return cuda_fail(s, r, "cudaGraphInstantiate");
    }
    r = cudaGraphLaunch(e->exec, s->stream);
    if (r) return cuda_fail(s, r, "cudaGraphLaunch");
    s->last_graph = 1;
  } else {
    r = enqueue_plan(s, e, s->stream);
    if (r) return cuda_fail(s, r, "fused pass launch");
  }
  std::memcpy(s->layout, e->layout_out.data(), sizeof(int) * s->n);
  s->last_passes = (int64_t)e->passes.size();
  s->last_launches = (int64_t)e->passes.size();
  s->last_relabels = e->relabels;
  s->last_k = e->tile_bits;
  s->last_blocks = e->fused_gates;
  s->last_jit = e->jit_state == 1 ? 1 : 0;
  s->last_flops_per_amp = e->flops_per_amp;
  return QC_OK;
}

qc_status run_unfused(qc_state* s, const qc_gate* ops, size_t n_ops, const MTable* mt) {
  int64_t launches = 0, relabels = 0;
  for (size_t i = 0; i < n_ops; ++i) {
    if (ops[i].op == QC_SWAP && s->relabel) {
      std::swap(s->layout[ops[i].qubits[0]], s->layout[ops[i].qubits[1]]);
      ++relabels;
      continue;
    }
    const PGate g = lower(ops[i], s->layout, mt);
    const int r = launch_gate(s->d, s->n, s->dbl, g, s->stream);
    if (r) return cuda_fail(s, r, "gate kernel launch");
    ++launches;
  }
  s->last_passes = launches;
  s->last_launches = launches;
  s->last_relabels = relabels;
  s->last_graph = 0;
  s->last_jit = 0;
  s->last_k = 0;
  return QC_OK;
}

qc_status ensure_stage(qc_state* s, size_t bytes) {
  if (s->stage_bytes >= bytes) return QC_OK;
  if (s->d_stage) cudaFree(s->d_stage);
  s->d_stage = nullptr;
  s->stage_bytes = 0;
  cudaError_t e = cudaMalloc(&s->d_stage, bytes);
  if (e != cudaSuccess) return fail(QC_ERR_OUT_OF_MEMORY, "staging buffer of %zu B: %s", bytes,
                                    cudaGetErrorString(e));
  s->stage_bytes = bytes;
  return QC_OK;
}

qc_status new_state(int n, qc_precision p, int device, void* stream, void* dev_ptr, qc_state** out,
                    int dist = 0, int world = 1, int rank = 0) {
  if (!out) return fail(QC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > kMaxQubits) return fail(QC_ERR_INVALID_ARG, "n=%d outside [1,%d]", n, kMaxQubits);
  if (p != QC_COMPLEX64 && p != QC_COMPLEX128) return fail(QC_ERR_INVALID_ARG, "bad precision %d", (int)p);
  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return fail(QC_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(QC_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  auto s = std::make_unique<qc_state>();
  s->n = n;
  s->prec = p;
  s->dbl = (p == QC_COMPLEX128);
  s->device = device;
  s->dist = dist;
  s->world = world;
  s->rank = rank;
  s->n_loc = n - std::countr_zero((unsigned)world);
  // loopback keeps every rank's shard in one buffer; NCCL keeps the local shard
  s->bytes = (size_t)(s->dbl ? 16 : 8) << (dist == 2 ? s->n_loc : n);
  canonical_layout(s.get());
  if (stream) {
    s->stream = reinterpret_cast<cudaStream_t>(stream);
  } else {
    e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(QC_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    s->own_stream = true;
  }
  if (dev_ptr) {
    if (reinterpret_cast<uintptr_t>(dev_ptr) % 16)
      return fail(QC_ERR_INVALID_ARG, "wrapped device pointer must be 16-byte aligned");
    s->d = dev_ptr;
  } else {
    e = cudaMalloc(&s->d, s->bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (s->own_stream) cudaStreamDestroy(s->stream);
      return fail(QC_ERR_OUT_OF_MEMORY, "cannot allocate the %d-qubit state: %zu bytes (%s)", n, s->bytes,
                  cudaGetErrorString(e));
    }
    s->own_mem = true;
    const int r = (dist == 2) ? launch_init_basis(s->d, s->n_loc, s->dbl, 0, s->stream) : launch_init_basis(s->d, n, s->dbl, 0, s->stream);
    if (r) {
      cudaFree(s->d);
      if (s->own_stream) cudaStreamDestroy(s->stream);
      return fail(QC_ERR_CUDA, "init: %s", cudaGetErrorString((cudaError_t)r));
    }
  }
  *out = s.release();
  return QC_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* qc_last_error(void) { return g_err.c_str(); }

const char* qc_version(void) { return "qc-b200 1 sm_100a"; }

qc_state* qc_state_create(int n, qc_precision p) {
  qc_state* s = nullptr;
  if (new_state(n, p, -1, nullptr, nullptr, &s) != QC_OK) return nullptr;
  return s;
}

qc_status qc_state_create_ex(int n, qc_precision p, int device, void* cuda_stream, qc_state** out) {
  if (device < 0) return fail(QC_ERR_INVALID_ARG, "device must be >= 0");
  return new_state(n, p, device, cuda_stream, nullptr, out);
}

qc_status qc_state_wrap(int n, qc_precision p, void* dev_ptr, void* cuda_stream, qc_state** out) {
  if (!dev_ptr) return fail(QC_ERR_INVALID_ARG, "dev_ptr is NULL");
  return new_state(n, p, -1, cuda_stream, dev_ptr, out);
}

qc_status qc_state_create_loopback(int n, qc_precision p, int world, qc_state** out) {
  if (world < 2 || (world & (world - 1)) || world > 64)
    return fail(QC_ERR_INVALID_ARG, "world must be a power of two in [2, 64]");
  if (n - std::countr_zero((unsigned)world) < 8)
    return fail(QC_ERR_INVALID_ARG, "each shard needs >= 8 local qubits");
  return new_state(n, p, -1, nullptr, nullptr, out, 1, world, 0);
}

qc_status qc_nccl_unique_id(void* out128) {
  if (!out128) return fail(QC_ERR_INVALID_ARG, "out is NULL");
  return nccl_get_unique_id(out128);
}

qc_status qc_state_create_dist(int n, qc_precision p, int rank, int world, const void* nccl_unique_id,
                               qc_state** out) {
  if (!out) return fail(QC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (world < 1 || (world & (world - 1)) || world > 64)
    return fail(QC_ERR_INVALID_ARG, "world must be a power of two in [1, 64]");
  if (rank < 0 || rank >= world) return fail(QC_ERR_INVALID_ARG, "rank out of range");
  if (world == 1) return new_state(n, p, -1, nullptr, nullptr, out);
  if (!nccl_unique_id) return fail(QC_ERR_INVALID_ARG, "nccl_unique_id is NULL");
  if (n - std::countr_zero((unsigned)world) < 8)
    return fail(QC_ERR_INVALID_ARG, "each shard needs >= 8 local qubits");
  qc_state* s = nullptr;
  qc_status st = new_state(n, p, -1, nullptr, nullptr, &s, 2, world, rank);
  if (st != QC_OK) return st;
  if (rank != 0) {  // |0...0> lives on rank 0 only
    cudaMemsetAsync(s->d, 0, s->bytes, s->stream);
  }
  st = nccl_create_comm(s, nccl_unique_id);
  if (st != QC_OK) {
    qc_state_destroy(s);
    return st;
  }
  *out = s;
  return QC_OK;
}

void qc_state_destroy(qc_state* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  s->plans.clear();
  dist_release(s);
  if (s->d_xstage) cudaFree(s->d_xstage);
  if (s->d_token) cudaFree(s->d_token);
  for (cudaEvent_t e : s->xev)
    if (e) cudaEventDestroy(e);
  if (s->xstream) cudaStreamDestroy(s->xstream);
  if (s->own_mem && s->d) cudaFree(s->d);
  if (s->d_stage) cudaFree(s->d_stage);
  if (s->d_partial) cudaFree(s->d_partial);
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->cstream) cudaStreamDestroy(s->cstream);
  for (cudaEvent_t e : s->cev)
    if (e) cudaEventDestroy(e);
  if (s->own_stream) cudaStreamDestroy(s->stream);
  delete s;
}

qc_status qc_state_init_basis(qc_state* s, uint64_t k) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if (k >> s->n) return fail(QC_ERR_INVALID_ARG, "basis index %llu >= 2^%d", (unsigned long long)k, s->n);
  canonical_layout(s);
  if (s->dist == 2) {  // canonical: rank r holds [r << n_loc, (r+1) << n_loc)
    const uint64_t nl = 1ull << s->n_loc;
    cudaError_t e = cudaMemsetAsync(s->d, 0, s->bytes, s->stream);
    if (e != cudaSuccess) return cuda_fail(s, e, "init_basis");
    if ((k / nl) == (uint64_t)s->rank) {  // the owning rank stores the single 1 at k mod 2^n_loc
      double one[2] = {1.0, 0.0};
      float onef[2] = {1.0f, 0.0f};
      e = cudaMemcpyAsync((char*)s->d + (k % nl) * amp_bytes(s), s->dbl ? (void*)one : (void*)onef,
                          amp_bytes(s), cudaMemcpyHostToDevice, s->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
      if (e != cudaSuccess) return cuda_fail(s, e, "init_basis");
    }
    return QC_OK;
  }
  const int r = launch_init_basis(s->d, s->n, s->dbl, k, s->stream);
  if (r) return cuda_fail(s, r, "init_basis");
  return QC_OK;
}

qc_status qc_state_init_random(qc_state* s, uint64_t seed) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  canonical_layout(s);
  const int r = (s->dist == 2) ? launch_init_random(s->d, s->n, s->dbl, seed, s->stream,
                                                   (uint64_t)s->rank << s->n_loc, 1ull << s->n_loc)
                               : launch_init_random(s->d, s->n, s->dbl, seed, s->stream);
  if (r) return cuda_fail(s, r, "init_random");
  return QC_OK;
}

qc_status qc_apply_gate(qc_state* s, qc_op op, const int* qubits, const double* matrix) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if ((int)op < 0 || (int)op > 15) return fail(QC_ERR_INVALID_ARG, "unknown op code %d", (int)op);
  if (!qubits) return fail(QC_ERR_INVALID_ARG, "qubits is NULL");
  qc_gate g;
  std::memset(&g, 0, sizeof g);
  g.op = op;
  for (int t = 0; t < kArity[op]; ++t) g.qubits[t] = qubits[t];
  g.ctrl_state = QC_CTRL_ONES;
  const bool has_theta = op == QC_P || op == QC_RX || op == QC_RY || op == QC_RZ || op == QC_CP;
  const int nm = op == QC_U2 ? 32 : ((op == QC_U1 || op == QC_CU1) ? 8 : 0);
  if ((has_theta || nm) && !matrix) return fail(QC_ERR_INVALID_ARG, "%s needs a matrix/theta argument", kName[op]);
  if (has_theta) g.theta = matrix[0];
  for (int i = 0; i < nm; ++i) g.m[i] = matrix[i];
  st = validate_gate(s->n, g, 0);
  if (st != QC_OK) return st;
  if (s->dist) return run_dist(s, &g, 1);
  return run_unfused(s, &g, 1, nullptr);
}

qc_status qc_apply_mgate(qc_state* s, const qc_mgate* mg) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if (!mg) return fail(QC_ERR_INVALID_ARG, "mgate is NULL");
  MTable mt(1);
  st = copy_mgate(s->n, *mg, 0, &mt[0]);
  if (st != QC_OK) return st;
  qc_gate g;
  std::memset(&g, 0, sizeof g);
  g.op = QC_MGATE;
  if (s->dist) return run_dist(s, &g, 1, &mt);
  return run_unfused(s, &g, 1, &mt);
}

qc_status qc_run_circuit_ex(qc_state* s, const qc_gate* ops, size_t n_ops, const qc_mgate* mgates,
                            size_t n_mgates) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if (n_ops && !ops) return fail(QC_ERR_INVALID_ARG, "ops is NULL");
  if (n_mgates && !mgates) return fail(QC_ERR_INVALID_ARG, "mgates is NULL");
  MTable table(n_mgates);
  for (size_t i = 0; i < n_mgates; ++i) {
    st = copy_mgate(s->n, mgates[i], i, &table[i]);
    if (st != QC_OK) return st;
  }
  const MTable* mt = n_mgates ? &table : nullptr;
  for (size_t i = 0; i < n_ops; ++i) {
    st = validate_gate(s->n, ops[i], i, mt);
    if (st != QC_OK) return st;
  }
  s->last_gates = (int64_t)n_ops;
  if (n_ops == 0) {
    s->last_passes = s->last_launches = s->last_relabels = 0;
    return QC_OK;
  }
  if (s->dist) return run_dist(s, ops, n_ops, mt);  // sharded: fused segments + exchanges
  if (s->fusion && s->n >= kSlotBits) return run_fused(s, ops, n_ops, mt);
  return run_unfused(s, ops, n_ops, mt);
}

qc_status qc_run_circuit(qc_state* s, const qc_gate* ops, size_t n_ops) {
  return qc_run_circuit_ex(s, ops, n_ops, nullptr, 0);
}

qc_status qc_state_sync(qc_state* s) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamSynchronize");
  return QC_OK;
}

qc_status qc_state_read(qc_state* s, uint64_t first, uint64_t count, void* host_dst) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  const uint64_t N = 1ull << s->n;
  if (!host_dst && count) return fail(QC_ERR_INVALID_ARG, "host_dst is NULL");
  if (first > N || count > N - first)
    return fail(QC_ERR_INVALID_ARG, "range [%llu,+%llu) exceeds 2^%d", (unsigned long long)first,
                (unsigned long long)count, s->n);
  if (!count) return QC_OK;
  if (s->dist == 2) {  // NCCL shard: canonical layout, range inside this rank's shard
    const uint64_t nl = 1ull << s->n_loc, lo = (uint64_t)s->rank * nl;
    if (!layout_is_canonical(s))
      return fail(QC_ERR_UNSUPPORTED, "sharded state: call qc_state_canonicalize (collective) first");
    if (first < lo || first + count > lo + nl)
      return fail(QC_ERR_INVALID_ARG, "sharded state: rank %d holds [%llu, %llu)", s->rank,
                  (unsigned long long)lo, (unsigned long long)(lo + nl));
    first -= lo;
  }
  const size_t ab = amp_bytes(s);
  cudaError_t e;
  if (layout_is_canonical(s)) {
    e = cudaMemcpyAsync(host_dst, (char*)s->d + first * ab, count * ab, cudaMemcpyDeviceToHost, s->stream);
    if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemcpyAsync D2H");
  } else {
    const uint64_t chunk = std::min<uint64_t>(count, (64ull << 20) / ab);
    st = ensure_stage(s, chunk * ab);
    if (st != QC_OK) return st;
    for (uint64_t c = 0; c < count; c += chunk) {
      const uint64_t m = std::min<uint64_t>(chunk, count - c);
      const int r = launch_gather(s->d, s->d_stage, s->n, s->dbl, s->layout, first + c, m, false, s->stream);
      if (r) return cuda_fail(s, r, "gather");
      e = cudaMemcpyAsync((char*)host_dst + c * ab, s->d_stage, m * ab, cudaMemcpyDeviceToHost, s->stream);
      if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemcpyAsync D2H");
    }
  }
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamSynchronize");
  return QC_OK;
}

qc_status qc_state_write(qc_state* s, uint64_t first, uint64_t count, const void* host_src) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  const uint64_t N = 1ull << s->n;
  if (!host_src && count) return fail(QC_ERR_INVALID_ARG, "host_src is NULL");
  if (first > N || count > N - first)
    return fail(QC_ERR_INVALID_ARG, "range [%llu,+%llu) exceeds 2^%d", (unsigned long long)first,
                (unsigned long long)count, s->n);
  if (!count) return QC_OK;
  if (s->dist == 2) {  // NCCL shard: canonical layout, range inside this rank's shard
    const uint64_t nl = 1ull << s->n_loc, lo = (uint64_t)s->rank * nl;
    if (!layout_is_canonical(s))
      return fail(QC_ERR_UNSUPPORTED, "sharded state: call qc_state_canonicalize (collective) first");
    if (first < lo || first + count > lo + nl)
      return fail(QC_ERR_INVALID_ARG, "sharded state: rank %d holds [%llu, %llu)", s->rank,
                  (unsigned long long)lo, (unsigned long long)(lo + nl));
    first -= lo;
  }
  const size_t ab = amp_bytes(s);
  cudaError_t e;
  if (layout_is_canonical(s)) {
    e = cudaMemcpyAsync((char*)s->d + first * ab, host_src, count * ab, cudaMemcpyHostToDevice, s->stream);
    if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemcpyAsync H2D");
  } else {
    const uint64_t chunk = std::min<uint64_t>(count, (64ull << 20) / ab);
    st = ensure_stage(s, chunk * ab);
    if (st != QC_OK) return st;
    for (uint64_t c = 0; c < count; c += chunk) {
      const uint64_t m = std::min<uint64_t>(chunk, count - c);
      e = cudaMemcpyAsync(s->d_stage, (const char*)host_src + c * ab, m * ab, cudaMemcpyHostToDevice, s->stream);
      if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemcpyAsync H2D");
      const int r = launch_gather(s->d, s->d_stage, s->n, s->dbl, s->layout, first + c, m, true, s->stream);
      if (r) return cuda_fail(s, r, "scatter");
    }
  }
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamSynchronize");
  return QC_OK;
}

// Read [first, first+count) into host_dst and write host_src in its place,
// chunk by chunk on two copy streams: the D2H of chunk c+1 (state stream)
// overlaps the H2D of chunk c (copy stream) -- PCIe is full duplex, so a
// result read-back and the next input upload take the time of one direction.
// Chunk c is written only after it has been read, so host_src == host_dst
// uploads exactly what was read.
qc_status qc_state_readwrite(qc_state* s, uint64_t first, uint64_t count, void* host_dst, const void* host_src) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  const uint64_t N = 1ull << s->n;
  if ((!host_dst || !host_src) && count) return fail(QC_ERR_INVALID_ARG, "host buffer is NULL");
  {
    const size_t nb = count * amp_bytes(s);
    const char *d0 = (const char*)host_dst, *s0 = (const char*)host_src;
    if (d0 != s0 && d0 < s0 + nb && s0 < d0 + nb)
      return fail(QC_ERR_INVALID_ARG, "host_dst and host_src overlap partially (must be identical or disjoint)");
  }
  if (first > N || count > N - first)
    return fail(QC_ERR_INVALID_ARG, "range [%llu,+%llu) exceeds 2^%d", (unsigned long long)first,
                (unsigned long long)count, s->n);
  if (!count) return QC_OK;
  if (!layout_is_canonical(s) && s->dist != 2) {  // gather / scatter path: one direction at a time
    st = qc_state_read(s, first, count, host_dst);
    return st == QC_OK ? qc_state_write(s, first, count, host_src) : st;
  }
  if (s->dist == 2) {
    const uint64_t nl = 1ull << s->n_loc, lo = (uint64_t)s->rank * nl;
    if (!layout_is_canonical(s))
      return fail(QC_ERR_UNSUPPORTED, "sharded state: call qc_state_canonicalize (collective) first");
    if (first < lo || first + count > lo + nl)
      return fail(QC_ERR_INVALID_ARG, "sharded state: rank %d holds [%llu, %llu)", s->rank,
                  (unsigned long long)lo, (unsigned long long)(lo + nl));
    first -= lo;
  }
  cudaError_t e = cudaSuccess;
  if (!s->cstream) {
    e = cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&s->cev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(s, e, "copy stream");
  }
  const size_t ab = amp_bytes(s);
  const uint64_t chunk = std::max<uint64_t>(1, (256ull << 20) / ab);
  char* dev = (char*)s->d + first * ab;
  for (uint64_t c = 0; c < count && e == cudaSuccess; c += chunk) {
    const size_t bytes = std::min<uint64_t>(chunk, count - c) * ab, off = c * ab;
    e = cudaMemcpyAsync((char*)host_dst + off, dev + off, bytes, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaEventRecord(s->cev[0], s->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s->cstream, s->cev[0], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dev + off, (const char*)host_src + off, bytes, cudaMemcpyHostToDevice, s->cstream);
  }
  if (e == cudaSuccess) e = cudaEventRecord(s->cev[1], s->cstream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, s->cev[1], 0);  // later work sees the upload
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "qc_state_readwrite");
  return QC_OK;
}

qc_status qc_state_canonicalize(qc_state* s) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if (s->dist) return dist_canonicalize(s);
  for (int q = 0; q < s->n; ++q) {
    const int want = s->n - 1 - q;
    if (s->layout[q] == want) continue;
    int q2 = -1;
    for (int u = 0; u < s->n; ++u)
      if (s->layout[u] == want) q2 = u;
    PGate g;
    g.kind = GK::SWAP2;
    g.t0 = s->layout[q];
    g.t1 = want;
    const int r = launch_gate(s->d, s->n, s->dbl, g, s->stream);
    if (r) return cuda_fail(s, r, "canonicalize");
    s->layout[q2] = s->layout[q];
    s->layout[q] = want;
  }
  return QC_OK;
}

qc_status qc_state_norm2(qc_state* s, double* out) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if (!out) return fail(QC_ERR_INVALID_ARG, "out is NULL");
  const int nb = sm_count() * 4;
  if (!s->d_partial) {
    cudaError_t e = cudaMalloc(&s->d_partial, nb * sizeof(double));
    if (e != cudaSuccess) return fail(QC_ERR_OUT_OF_MEMORY, "norm partials: %s", cudaGetErrorString(e));
  }
  const int r = launch_norm2(s->d, s->dist == 2 ? s->n_loc : s->n, s->dbl, s->d_partial, nb, s->stream);
  if (r) return cuda_fail(s, r, "norm2");
  std::vector<double> h(nb);
  cudaError_t e = cudaMemcpyAsync(h.data(), s->d_partial, nb * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemcpyAsync");
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamSynchronize");
  double t = 0;
  for (double v : h) t += v;
  if (s->dist == 2) {
    st = nccl_allreduce_sum(s, &t);
    if (st != QC_OK) return st;
  }
  *out = t;
  return QC_OK;
}

qc_status qc_set_option(qc_state* s, qc_option opt, int64_t v) {
  if (!s) return fail(QC_ERR_INVALID_ARG, "state is NULL");
  switch (opt) {
    case QC_OPT_FUSION: s->fusion = v != 0; break;
    case QC_OPT_RELABEL_SWAP: s->relabel = v != 0; break;
    case QC_OPT_USE_GRAPH: s->use_graph = v != 0; break;
    case QC_OPT_TILE_BITS:
      if (v != 0 && (v < 4 || v > 13)) return fail(QC_ERR_INVALID_ARG, "tile bits must be 0 or 4..13");
      s->tile_bits = (int)v;
      break;
    case QC_OPT_CTAS:
      if (v < 0 || v > 65535) return fail(QC_ERR_INVALID_ARG, "ctas out of range");
      s->ctas = (int)v;
      break;
    case QC_OPT_BLOCK_FUSION: s->block_fusion = v != 0; break;
    case QC_OPT_ROW_BITS:
      if (v != 0 && (v < 1 || v > 11)) return fail(QC_ERR_INVALID_ARG, "row bits must be 0 or 1..11");
      s->row_bits = (int)v;
      break;
    case QC_OPT_TMA_MODE:
      if (v < 0 || v > 2) return fail(QC_ERR_INVALID_ARG, "tma mode must be 0, 1 or 2");
      s->tma_mode = (int)v;
      break;
    case QC_OPT_REMAP: s->remap = v != 0; break;
    case QC_OPT_EXCHANGE:
      if (v < 0 || v > 3)
        return fail(QC_ERR_INVALID_ARG, "exchange must be 0 (NCCL), 1 (P2P), 2 (pair passes) or 3 (group plan)");
      s->xmode = (int)v;
      break;
    case QC_OPT_JIT:
      if (v < 0 || v > 2) return fail(QC_ERR_INVALID_ARG, "jit must be 0, 1 or 2");
      s->jit = (int)v;
      break;
    default: return fail(QC_ERR_INVALID_ARG, "unknown option %d", (int)opt);
  }
  return QC_OK;
}

qc_status qc_get_info(const qc_state* s, qc_info* out) {
  if (!s || !out) return fail(QC_ERR_INVALID_ARG, "NULL argument");
  std::memset(out, 0, sizeof *out);
  out->n = s->n;
  out->precision = s->prec;
  out->device_ptr = s->d;
  out->stream = s->stream;
  for (int q = 0; q < s->n; ++q) out->layout[q] = s->layout[q];
  out->layout_is_canonical = layout_is_canonical(s) ? 1 : 0;
  out->last_gates = s->last_gates;
  out->last_passes = s->last_passes;
  out->last_launches = s->last_launches;
  out->last_relabels = s->last_relabels;
  out->last_graph = s->last_graph;
  out->tile_bits = s->last_k;
  out->last_blocks = s->last_blocks;
  out->last_jit = s->last_jit;
  out->world = s->world;
  out->rank = s->rank;
  out->n_local = s->dist ? s->n_loc : s->n;
  out->sharding = s->dist;
  out->last_exchanges = s->last_exchanges;
  out->last_pair_segments = s->last_pair_segments;
  out->last_flops_per_amp = s->last_flops_per_amp;
  return QC_OK;
}

}  // extern "C"

extern "C" qc_status qc_debug_plan(int n, qc_precision p, const qc_gate* ops, size_t n_ops, int tile_bits,
                                   int row_bits, int block_fusion, int remap, int compile_jit, qc_plan_stats* out,
                                   char* errbuf, size_t errlen) {
  auto err = [&](qc_status st, const std::string& m) {
    fail(st, "%s", m.c_str());
    if (errbuf && errlen) snprintf(errbuf, errlen, "%s", m.c_str());
    return st;
  };
  if (!out) return err(QC_ERR_INVALID_ARG, "out is NULL");
  std::memset(out, 0, sizeof *out);
  if (n < 1 || n > kMaxQubits) return err(QC_ERR_INVALID_ARG, "bad n");
  if (n_ops && !ops) return err(QC_ERR_INVALID_ARG, "ops is NULL");
  for (size_t i = 0; i < n_ops; ++i)
    if (validate_gate(n, ops[i], i) != QC_OK) return err(QC_ERR_INVALID_ARG, g_err);
  const bool dbl = p == QC_COMPLEX128;
  int k = tile_bits ? tile_bits : (dbl ? 12 : 13);
  if (dbl && k > 12) k = 12;
  if (k > n) k = n;
  int rb = row_bits ? row_bits : (dbl ? 6 : 7);
  if (rb > k - 2) rb = k - 2;
  if (rb < 1) rb = 1;
  int lay[64];
  for (int q = 0; q < n; ++q) lay[q] = n - 1 - q;
  std::vector<PGate> gates;
  for (size_t i = 0; i < n_ops; ++i) {
    if (ops[i].op == QC_SWAP) {
      std::swap(lay[ops[i].qubits[0]], lay[ops[i].qubits[1]]);
      out->relabels++;
      continue;
    }
    gates.push_back(lower(ops[i], lay));
  }
  out->gates = (int64_t)n_ops;
  out->tile_bits = k;
  std::vector<PGate> blocks = block_fusion ? fuse_blocks(gates, ~0ull) : gates;
  out->blocks = (int64_t)blocks.size();
  if (blocks.empty()) return QC_OK;
  FusedPlan fp = plan_best(n, k, rb, row_bits, true, dbl, blocks, remap != 0, &rb);  // default transport
  if (!fp.ok) return err(QC_ERR_UNSUPPORTED, "planner failed");
  out->remap_swaps = fp.remap_swaps;
  out->flops_per_amp = plan_flops_per_amp(fp);
  out->restore_passes = fp.restore_passes;
  // mirror build_fused_entry's layout choice (boxes, else make_row_tmap's gather4 limits)
  const bool g4 = ((uint64_t)(dbl ? 16 : 8) << rb) <= 1024 && n - rb <= 31 && n - rb >= 2;
  for (auto& pp : fp.passes) {
    pp.desc.g4 = g4 ? 1 : 0;
    pp.desc.pshift = g4 ? 31 : rb;
    if (make_box_tmap(nullptr, n, dbl, pass_tile_set(pp.desc), nullptr, &pp.desc)) {
      pp.desc.g4 = 2;
      pp.desc.pshift = 31;
    }
  }
  out->passes = (int64_t)fp.passes.size();
  const int LB = dbl ? 3 : 4;  // tile bits inside one 16-B / 8-B bank-group phase (jit.cu)
  for (auto& pp : fp.passes) {
    for (auto& sd : pp.subs) {
      int x = 0;
      for (int j = 0; j < kSlotBits; ++j) x += sd.g[j] < LB;
      out->swz_substages += x >= 2;
    }
    out->substages += (int64_t)pp.subs.size();
    out->fused_ops += (int64_t)pp.ops.size();
    for (auto& o : pp.ops) out->phase_runs += o.h.kind == F_PRUN;
  }
  std::vector<uint8_t> blob = pack_plan(fp, dbl);
  out->blob_bytes = (int64_t)blob.size();
  if (compile_jit) {
    std::string e;
    int compiled = 0;
    if (!jit_compile_only(fp, dbl, compiled, e)) return err(QC_ERR_UNSUPPORTED, e);
    out->jit_compiled = compiled;
  }
  return QC_OK;
}

extern "C" qc_status qc_debug_exchange_runs(int n_loc, int rank, int g, int l, int* partner, uint64_t* offsets,
                                           uint64_t* counts, int max_runs, int* n_runs) {
  if (!partner || !n_runs || g < n_loc || l < 0 || l >= n_loc) return fail(QC_ERR_INVALID_ARG, "bad arguments");
  const auto runs = exchange_runs(n_loc, rank, g, l, partner);
  *n_runs = (int)runs.size();
  for (int i = 0; i < (int)runs.size() && i < max_runs; ++i) {
    if (offsets) offsets[i] = runs[i].offset;
    if (counts) counts[i] = runs[i].count;
  }
  return QC_OK;
}

extern "C" qc_status qc_debug_dist_schedule(int n, int world, int relabel, const qc_gate* ops, size_t n_ops,
                                           int* steps, int max_steps, int* n_steps, int* layout_out) {
  return qc_debug_dist_schedule_ex(n, world, relabel, 0, ops, n_ops, steps, max_steps, n_steps, layout_out);
}

extern "C" qc_status qc_debug_dist_schedule_ex(int n, int world, int relabel, int exchange_mode, const qc_gate* ops,
                                              size_t n_ops, int* steps, int max_steps, int* n_steps,
                                              int* layout_out) {
  if (exchange_mode < 0 || exchange_mode > 3) return fail(QC_ERR_INVALID_ARG, "bad exchange mode");
  if (!n_steps || world < 2 || (world & (world - 1))) return fail(QC_ERR_INVALID_ARG, "bad arguments");
  for (size_t i = 0; i < n_ops; ++i) {
    const qc_status st = validate_gate(n, ops[i], i);
    if (st != QC_OK) return st;
  }
  std::vector<int> out, lay;
  const qc_status st = dist_schedule_dry(n, world, relabel, ops, n_ops, out, lay, nullptr, exchange_mode);
  if (st != QC_OK) return st;
  *n_steps = (int)out.size() / 4;
  if (steps) std::memcpy(steps, out.data(), sizeof(int) * std::min<size_t>(out.size(), (size_t)max_steps * 4));
  if (layout_out) std::memcpy(layout_out, lay.data(), sizeof(int) * lay.size());
  return QC_OK;
}

extern "C" qc_status qc_debug_group_split(int n, int world, uint64_t tile_bits_set, int rank, uint64_t* tile0,
                                         uint64_t* count, int* j, int* owners) {
  if (world < 2 || (world & (world - 1)) || n < 2 || n > 62 || rank < 0 || rank >= world || !tile0 || !count ||
      !j || !owners)
    return fail(QC_ERR_INVALID_ARG, "bad arguments");
  const int p = std::countr_zero((unsigned)world), nl = n - p, k = std::popcount(tile_bits_set);
  if ((tile_bits_set >> n) || k > nl || nl < 1) return fail(QC_ERR_INVALID_ARG, "bad tile bit set");
  const GroupSplit sp = group_split(nl, p, tile_bits_set, 1ull << (n - k), rank);
  *tile0 = sp.tile0;
  *count = sp.count;
  *j = sp.j;
  for (int h = 0; h < 8; ++h) owners[h] = sp.owner[h];
  return QC_OK;
}

extern "C" qc_status qc_debug_exchange(qc_state* s, int g, int l) {
  qc_status st = check_state(s);
  if (st != QC_OK) return st;
  if (!s->dist) return fail(QC_ERR_INVALID_ARG, "state is not sharded");
  if (g < s->n_loc || g >= s->n || l < 0 || l >= s->n_loc) return fail(QC_ERR_INVALID_ARG, "bad bits");
  st = dist_exchange(s, g, l);
  if (st != QC_OK) return st;
  // the data now has physical bits g and l swapped: keep the layout truthful
  for (int q = 0; q < s->n; ++q) {
    if (s->layout[q] == g) s->layout[q] = l;
    else if (s->layout[q] == l) s->layout[q] = g;
  }
  return QC_OK;
}

extern "C" qc_status qc_debug_box_layout(uint64_t T, int nbits, int dbl, int* dims, int* starts, int* boxbits,
                                         uint32_t* xmask) {
  if (!dims || !starts || !boxbits || !xmask) return fail(QC_ERR_INVALID_ARG, "NULL argument");
  if (nbits < 1 || nbits > 62 || (T >> nbits)) return fail(QC_ERR_INVALID_ARG, "bad tile set");
  PassDesc d{};
  if (!make_box_tmap(nullptr, nbits, dbl != 0, T, nullptr, &d)) return fail(QC_ERR_UNSUPPORTED, "no box layout");
  *dims = d.bx_dims;
  for (int i = 0; i <= d.bx_dims; ++i) starts[i] = d.bx_start[i];
  for (int i = 0; i < d.bx_dims; ++i) {
    const uint64_t in_dim = ((T >> d.bx_start[i]) & ((1ull << (d.bx_start[i + 1] - d.bx_start[i])) - 1));
    boxbits[i] = std::countr_one(in_dim);
  }
  *xmask = d.bx_xmask;
  return QC_OK;
}

extern "C" qc_status qc_debug_fma_peak(int dbl, double* tflops) {
  if (!tflops) return fail(QC_ERR_INVALID_ARG, "tflops is NULL");
  const int r = fma_peak(dbl != 0, tflops);
  if (r) return fail(QC_ERR_CUDA, "fma peak kernel: %s", cudaGetErrorString((cudaError_t)r));
  return QC_OK;
}
