// plan.cpp -- fusion planner: lowered gates -> fused tile passes.
//
// Greedy in-order scheduling (hard part 1): a pass starts with the
// row bits 0..rb-1 in its tile set T.  Walking the remaining gates in order,
// a gate joins the pass when (a) it shares no qubit with any gate already
// deferred from this pass (so moving it ahead of them is a commutation of
// disjoint operators, exact) and (b) its non-diagonal targets fit in T with
// |T| <= k.  Diagonal gates and control bits never need to be in T (their
// bit values are per-tile or per-task constants).  A gate that does not join
// is deferred and blocks its qubits.  Within a pass, consecutive gates are
// cut into sub-stages whose non-diagonal targets fit in a 4-bit slot group.
// Every gate is applied exactly once, and the relative order of gates that
// share a qubit is preserved, so the product of the passes is the circuit
// (eq:kron composed in order).
#include <algorithm>
#include <bit>
#include <cstring>

#include "qc_internal.h"

namespace qc {
namespace {

inline int popc(uint64_t x) { return std::popcount(x); }

uint64_t target_mask(const PGate& g) {
  uint64_t m = 1ull << g.t0;
  if (g.kind == GK::DENSE2 || g.kind == GK::SWAP2) m |= 1ull << g.t1;
  return m;
}
uint64_t need_mask(const PGate& g) { return g.kind == GK::DIAG1 ? 0ull : target_mask(g); }

struct Frame {
  uint64_t T;                 // tile bits (physical)
  int local_of[64];           // physical -> tile-local position (-1 outside)
  int n_local;
};

Frame make_frame(int n, int rb, uint64_t T) {
  Frame f{};
  f.T = T;
  for (int p = 0; p < 64; ++p) f.local_of[p] = -1;
  int l = 0;
  for (int p = 0; p < rb; ++p) f.local_of[p] = l++;
  for (int p = rb; p < n; ++p)
    if (T & (1ull << p)) f.local_of[p] = l++;
  f.n_local = l;
  return f;
}

void encode_op(const PGate& g, const Frame& f, const int slot_of_local[64], FOpT<double>& o) {
  std::memset(&o, 0, sizeof(o));
  auto slot_of = [&](int p) { return f.local_of[p] >= 0 ? slot_of_local[f.local_of[p]] : -1; };
  switch (g.kind) {
    case GK::DENSE1: o.kind = F_DENSE1; o.sb0 = slot_of(g.t0); break;
    case GK::PERM1: o.kind = F_PERM1; o.sb0 = slot_of(g.t0); break;
    case GK::DENSE2: o.kind = F_DENSE2; o.sb0 = slot_of(g.t0); o.sb1 = slot_of(g.t1); break;
    case GK::SWAP2: {
      o.kind = F_SWAP2;
      const int a = slot_of(g.t0), b = slot_of(g.t1);
      o.sb0 = std::min(a, b);
      o.sb1 = std::max(a, b);
      break;
    }
    case GK::DIAG1: {
      o.kind = F_DIAG1;
      const int s = slot_of(g.t0);
      if (s >= 0) {
        o.dsrc = D_SLOT;
        o.sb0 = s;
      } else if (f.local_of[g.t0] >= 0) {
        o.dsrc = D_LOCAL;
        o.dbit = f.local_of[g.t0];
      } else {
        o.dsrc = D_OUTER;
        o.dbit = g.t0;
      }
      o.d0_is_one = g.d0_is_one ? 1 : 0;
      break;
    }
  }
  for (int p = 0; p < 64; ++p) {
    if (!(g.cmask & (1ull << p))) continue;
    const uint64_t want = (g.cval >> p) & 1ull;
    const int s = slot_of(p);
    if (s >= 0) {
      o.smask |= 1u << s;
      o.sval |= (uint32_t)want << s;
    } else if (f.local_of[p] >= 0) {
      o.lmask |= 1u << f.local_of[p];
      o.lval |= (uint32_t)want << f.local_of[p];
    } else {
      o.omask |= 1ull << p;
      o.oval |= want << p;
    }
  }
  const int nm = (g.kind == GK::DENSE2) ? 16 : 4;
  for (int i = 0; i < nm; ++i) {
    o.m[2 * i] = g.m[i].real();
    o.m[2 * i + 1] = g.m[i].imag();
  }
}

}  // namespace

FusedPlan plan_fused(int n, int k, int rb, const std::vector<PGate>& gates) {
  FusedPlan plan;
  std::vector<int> remaining(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) remaining[i] = (int)i;
  const uint64_t all_bits = (n >= 64) ? ~0ull : ((1ull << n) - 1);

  while (!remaining.empty()) {
    uint64_t T = (1ull << rb) - 1;
    uint64_t blocked = 0;
    std::vector<int> taken, deferred;
    for (int gi : remaining) {
      const PGate& g = gates[gi];
      if (popc(need_mask(g)) + rb > k && n > k) {  // cannot happen when rb <= k-2
        plan.ok = false;
        return plan;
      }
      const uint64_t all = target_mask(g) | g.cmask;
      if (all & blocked) {
        blocked |= all;
        deferred.push_back(gi);
        continue;
      }
      const uint64_t nt = T | need_mask(g);
      if (popc(nt) <= k) {
        T = nt;
        taken.push_back(gi);
      } else {
        blocked |= all;
        deferred.push_back(gi);
      }
    }
    // Fill T to k bits with the lowest free bits (longer contiguous runs).
    for (int p = rb; popc(T) < k && p < n; ++p) T |= 1ull << p;
    (void)all_bits;

    FusedPassPlan pp{};
    const Frame f = make_frame(n, rb, T);
    PassDesc& d = pp.desc;
    d.k = k;
    d.rb = rb;
    d.n_hi = 0;
    for (int p = rb; p < n; ++p)
      if (T & (1ull << p)) d.hi_pos[d.n_hi++] = p;
    d.n_outer = 0;
    for (int p = 0; p < n; ++p)
      if (!(T & (1ull << p))) d.outer_pos[d.n_outer++] = p;
    d.n_tiles = 1ull << (n - k);
    d.sub_begin = (int)plan.subs.size();
    pp.gate_ids = taken;

    // ---- sub-stages: consecutive gates whose targets fit a 4-bit slot group
    size_t gi = 0;
    while (gi < taken.size()) {
      uint64_t G = 0;
      size_t gj = gi;
      while (gj < taken.size()) {
        const uint64_t ng = G | need_mask(gates[taken[gj]]);
        if (popc(ng) > kSlotBits) break;
        G = ng;
        ++gj;
      }
      // pad G with the highest tile-local bits (keeps lanes on contiguous rows)
      int glocal[kSlotBits];
      int ng = 0;
      bool in_g[64] = {false};
      for (int p = 0; p < n; ++p)
        if (G & (1ull << p)) in_g[f.local_of[p]] = true;
      int cnt = popc(G);
      for (int l = f.n_local - 1; l >= 0 && cnt < kSlotBits; --l) {
        if (in_g[l]) continue;
        in_g[l] = true;
        ++cnt;
      }
      for (int l = 0; l < f.n_local; ++l)
        if (in_g[l]) glocal[ng++] = l;
      SubStageDesc sd{};
      int slot_of_local[64];
      for (int l = 0; l < 64; ++l) slot_of_local[l] = -1;
      for (int j = 0; j < kSlotBits; ++j) {
        sd.g[j] = glocal[j];
        slot_of_local[glocal[j]] = j;
      }
      sd.op_begin = (int)plan.ops.size();
      for (size_t x = gi; x < gj; ++x) {
        FOpT<double> o;
        encode_op(gates[taken[x]], f, slot_of_local, o);
        plan.ops.push_back(o);
      }
      sd.op_end = (int)plan.ops.size();
      plan.subs.push_back(sd);
      gi = gj;
    }
    d.sub_end = (int)plan.subs.size();
    plan.passes.push_back(pp);
    remaining.swap(deferred);
  }
  return plan;
}

}  // namespace qc
