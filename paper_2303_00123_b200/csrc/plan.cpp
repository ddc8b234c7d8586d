// plan.cpp -- fusion planner: (fused) gate blocks -> fused tile passes.
//
// Greedy in-order scheduling (hard part 1): a pass starts with the
// row bits 0..rb-1 in its tile set T.  Walking the remaining gates in order,
// a gate joins the pass when (a) it shares no bit with any gate already
// deferred from this pass (so moving it ahead of them is a commutation of
// operators on disjoint bits -- exact) and (b) its non-diagonal targets fit
// in T with |T| <= k.  Diagonal gates and control bits never need to be in T
// (their bit values are per-tile or per-task constants).  A gate that does
// not join is deferred and blocks its bits.  Within a pass, consecutive gates
// are cut into sub-stages whose non-diagonal targets fit a 4-bit slot group;
// runs of consecutive phase gates sharing a bit (e.g. the controlled-phase
// ladder after each Hadamard of the QFT) become one "phase run"
// whose factors from bits outside the tile are evaluated once per tile.
// Every gate is applied exactly once and gates sharing a bit keep their
// order, so the product of the passes is the circuit (eq:kron in order).
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "qc_internal.h"

namespace qc {
namespace {

inline int popc(uint64_t x) { return std::popcount(x); }

uint64_t target_mask(const PGate& g) { return pgate_targets(g); }
uint64_t need_mask(const PGate& g) { return g.kind == GK::DIAG1 ? 0ull : target_mask(g); }

// Algorithmic flops per state amplitude of one (block-fused) gate inside a
// fused pass, as plan_flops_per_amp counts them (complex multiply 6, multiply-
// accumulate 8), halved per control bit.  Used for the per-pass FP64 budget.
double gate_flops(const PGate& g) {
  const double ctrl = std::ldexp(1.0, -popc(g.cmask));
  switch (g.kind) {
    case GK::DENSE1: return 14 * ctrl;
    case GK::DIAG1: return (g.d0_is_one ? 3 : 6) * ctrl;
    case GK::DENSE2: return 30 * ctrl;
    case GK::SPARSE2: return 14 * ctrl;
    case GK::DIAG2: return 6 * ctrl;
    case GK::DENSEK: return (6.0 + 8.0 * ((1 << g.nt) - 1)) * ctrl;
    default: return 0;  // permutations / swaps: register moves
  }
}

size_t blob_estimate(const PGate& g) {
  if (g.kind == GK::DIAG1) return 48;
  if (g.kind == GK::DENSEK) return 48 + ((size_t)16 << (2 * g.nt));
  if (pgate_is_two(g)) return 48 + 16 * 16;
  return 48 + 4 * 16;
}

struct Frame {
  int local_of[64];  // physical -> tile-local position (-1 outside)
  int n_local;
};

Frame make_frame(int n, int rb, uint64_t T) {
  Frame f{};
  for (int p = 0; p < 64; ++p) f.local_of[p] = -1;
  int l = 0;
  for (int p = 0; p < rb; ++p) f.local_of[p] = l++;
  for (int p = rb; p < n; ++p)
    if (T & (1ull << p)) f.local_of[p] = l++;
  f.n_local = l;
  return f;
}

struct Ctx {
  const Frame* f;
  int slot_of_local[64];
  int slot(int p) const { return f->local_of[p] >= 0 ? slot_of_local[f->local_of[p]] : -1; }
  uint8_t src(int p) const {
    if (slot(p) >= 0) return S_SLOT;
    return f->local_of[p] >= 0 ? S_LOCAL : S_OUTER;
  }
  uint8_t bitpos(int p) const {  // slot bit / local position / physical bit
    const int s = slot(p);
    if (s >= 0) return (uint8_t)s;
    return (uint8_t)(f->local_of[p] >= 0 ? f->local_of[p] : p);
  }
};

void set_pred(FHdr& h, const PGate& g, const Ctx& c) {
  for (int p = 0; p < 64; ++p) {
    if (!(g.cmask & (1ull << p))) continue;
    const uint64_t want = (g.cval >> p) & 1ull;
    const int s = c.slot(p);
    if (s >= 0) {
      h.smask |= (uint8_t)(1u << s);
      h.sval |= (uint8_t)(want << s);
    } else if (c.f->local_of[p] >= 0) {
      h.lmask |= 1u << c.f->local_of[p];
      h.lval |= (uint32_t)want << c.f->local_of[p];
    } else {
      h.omask |= 1ull << p;
      h.oval |= want << p;
    }
  }
}

bool is0(cd z) { return z.real() == 0.0 && z.imag() == 0.0; }
bool is1(cd z) { return z.real() == 1.0 && z.imag() == 0.0; }

// Exact structure of a 2x2 / 4x4 matrix -> kernel pattern + coefficients.
void rows_to_ir(const cd* M, int dim, FOpIR& o) {
  bool diag = true, perm = true;
  for (int r = 0; r < dim; ++r) {
    int nnz = 0;
    for (int c = 0; c < dim; ++c) {
      const cd v = M[r * dim + c];
      if (r != c && !is0(v)) diag = false;
      if (!is0(v)) {
        ++nnz;
        if (!is1(v)) perm = false;
      }
    }
    if (nnz != 1) perm = false;
  }
  o.h.identmask = 0;
  if (diag) {
    o.h.dsrc = P_DIAG;
    for (int r = 0; r < dim; ++r)
      if (is1(M[r * dim + r])) o.h.identmask |= (uint8_t)(1u << r);
    for (int r = 0; r < dim; ++r)
      if (dim == 4 || !(o.h.identmask & (1u << r))) o.coefs.push_back(M[r * dim + r]);
    return;
  }
  if (perm) {
    o.h.dsrc = P_MOVE;
    for (int r = 0; r < dim; ++r)
      for (int c = 0; c < dim; ++c)
        if (is1(M[r * dim + c])) o.h.nz[r] = (uint8_t)c;
    return;
  }
  if (dim == 2) {
    if (is0(M[0]) && is0(M[3])) {
      o.h.dsrc = P_ANTI;
      o.coefs = {M[1], M[2]};
    } else {
      o.h.dsrc = P_DENSE;
      o.coefs = {M[0], M[1], M[2], M[3]};
    }
    return;
  }
  for (int X = 1; X <= 3; ++X) {
    bool ok = true;
    for (int r = 0; r < 4 && ok; ++r)
      for (int c = 0; c < 4; ++c)
        if (c != r && c != (r ^ X) && !is0(M[4 * r + c])) ok = false;
    if (!ok) continue;
    o.h.dsrc = (uint8_t)(P_PAIRS1 + X - 1);
    for (int r = 0; r < 4; ++r) {
      o.coefs.push_back(M[4 * r + r]);
      o.coefs.push_back(M[4 * r + (r ^ X)]);
      if (is1(M[4 * r + r]) && is0(M[4 * r + (r ^ X)])) o.h.identmask |= (uint8_t)(1u << r);
    }
    return;
  }
  o.h.dsrc = P_DENSE;
  for (int i = 0; i < 16; ++i) o.coefs.push_back(M[i]);
}

// Generic k-target gate (k = 3, 4) -> F_MK in canonical slot order: the
// listed targets' slot bits s_j; matrix index bit i of the canonical form is
// the i-th lowest of {s_j}, so M'[perm(r)][perm(c)] = M[r][c] (a relabelling
// of the same operator's index bits).
FOpIR convert_mk(const PGate& g, const Ctx& c) {
  FOpIR o;
  set_pred(o.h, g, c);
  o.h.kind = F_MK;
  const int k = g.nt, d = 1 << k;
  int sl[4], rank[4];
  unsigned present = 0;
  for (int j = 0; j < k; ++j) {
    sl[j] = c.slot(g.tk[j]);
    present |= 1u << sl[j];
  }
  for (int j = 0; j < k; ++j) {  // rank of s_j among the op's slot bits (0 = lowest)
    rank[j] = 0;
    for (int i = 0; i < k; ++i) rank[j] += sl[i] < sl[j];
  }
  o.h.sb1 = (uint8_t)k;
  o.h.sb0 = 0;
  if (k == 3)
    for (int b = 0; b < kSlotBits; ++b)
      if (!(present & (1u << b))) o.h.sb0 = (uint8_t)b;
  auto perm = [&](int r) {  // listed index (target j = bit k-1-j) -> canonical index
    int x = 0;
    for (int j = 0; j < k; ++j)
      if ((r >> (k - 1 - j)) & 1) x |= 1 << rank[j];
    return x;
  };
  o.mk.assign((size_t)d * d, cd(0));
  for (int r = 0; r < d; ++r)
    for (int cc = 0; cc < d; ++cc) o.mk[(size_t)perm(r) * d + perm(cc)] = (*g.mk)[(size_t)r * d + cc];
  o.coefs = o.mk;
  return o;
}

// A single (non-run) gate -> one fused op.
FOpIR convert(const PGate& g, const Ctx& c) {
  if (g.kind == GK::DENSEK) return convert_mk(g, c);
  FOpIR o;
  set_pred(o.h, g, c);
  if (pgate_is_two(g)) {
    o.h.kind = F_M2;
    o.h.sb0 = (uint8_t)c.slot(g.t0);
    o.h.sb1 = (uint8_t)c.slot(g.t1);
    cd M[16];
    pgate_dense4(g, M);
    rows_to_ir(M, 4, o);
    for (int i = 0; i < 16; ++i) o.dense[i] = M[i];
    return o;
  }
  cd M[4] = {0, 0, 0, 0};
  switch (g.kind) {
    case GK::DENSE1: for (int i = 0; i < 4; ++i) M[i] = g.m[i]; break;
    case GK::PERM1: M[1] = 1; M[2] = 1; break;
    default: M[0] = g.m[0]; M[3] = g.m[1]; break;  // DIAG1
  }
  if (g.kind == GK::DIAG1 && c.slot(g.t0) < 0) {
    o.h.kind = F_DSCALE;
    o.h.dsrc = c.src(g.t0);
    o.h.dbit = c.bitpos(g.t0);
    o.h.flags = g.d0_is_one ? 1 : 0;
    o.coefs = {g.m[0], g.m[1]};
    return o;
  }
  o.h.kind = F_M1;
  o.h.sb0 = (uint8_t)c.slot(g.t0);
  rows_to_ir(M, 2, o);
  for (int i = 0; i < 4; ++i) o.dense[i] = M[i];
  return o;
}

// Within one pass every amplitude of a tile sees every unpredicated op once,
// and scalars commute with everything: pull a common real magnitude c out of
// each unpredicated M op (the Hadamards' 1/sqrt2, making H blocks +-1
// additions) and fold the product into the pass's first unpredicated M op.
void factor_pass_scalars(FusedPassPlan& pp) {
  FOpIR* first = nullptr;
  double C = 1.0;
  for (auto& o : pp.ops) {
    if (o.h.kind != F_M1 && o.h.kind != F_M2) continue;
    if (o.h.smask || o.h.lmask || o.h.omask) continue;
    if (o.h.dsrc == P_MOVE) continue;  // permutations stay pure moves
    const int dim = o.h.kind == F_M1 ? 2 : 4;
    if (!first) {
      first = &o;
      continue;
    }
    double c = 0;
    bool ok = true;
    for (int i = 0; i < dim * dim && ok; ++i) {
      const double m = std::abs(o.dense[i]);
      if (m == 0) continue;
      if (c == 0) c = m;
      else if (std::fabs(m - c) > 1e-14 * c) ok = false;
    }
    if (!ok || c == 0 || c == 1.0) continue;
    for (int i = 0; i < dim * dim; ++i) o.dense[i] /= c;
    C *= c;
    o.coefs.clear();
    o.h.identmask = 0;
    rows_to_ir(o.dense, dim, o);
  }
  if (first && C != 1.0) {
    const int dim = first->h.kind == F_M1 ? 2 : 4;
    for (int i = 0; i < dim * dim; ++i) first->dense[i] *= C;
    first->coefs.clear();
    first->h.identmask = 0;
    rows_to_ir(first->dense, dim, *first);
  }
}

bool phase_type(const PGate& g) { return g.kind == GK::DIAG1 && popc(g.cmask) <= 1; }

uint64_t base_cands(const PGate& g) {
  uint64_t m = 1ull << g.t0;
  if (g.cmask && g.d0_is_one && (g.cval & g.cmask) == g.cmask) m |= g.cmask;  // symmetric CP
  return m;
}

// Phase run over gates [i, j) of `seq` with common bit `base`.
void emit_run(const std::vector<PGate>& seq, size_t i, size_t j, int base, const Ctx& c,
              int& n_prun, std::vector<FOpIR>& out) {
  FOpIR run;
  run.h.kind = F_PRUN;
  run.h.dsrc = c.src(base);
  if (run.h.dsrc == S_SLOT)
    run.h.sb0 = (uint8_t)c.slot(base);
  else
    run.h.dbit = c.bitpos(base);
  std::vector<FOpIR::Term> loc, outer, none;
  bool any0 = false;
  std::vector<FOpIR> extra;
  for (size_t x = i; x < j; ++x) {
    const PGate& g = seq[x];
    FOpIR::Term t{};
    int ctrl = -1;
    uint8_t cval = 1;
    if (g.t0 == base) {
      t.d0 = g.m[0];
      t.d1 = g.m[1];
      if (g.cmask) {
        ctrl = std::countr_zero(g.cmask);
        cval = (uint8_t)((g.cval >> ctrl) & 1ull);
      }
    } else {  // symmetric CP with base = its control: phase iff target = 1
      ctrl = g.t0;
      cval = 1;
      t.d0 = 1;
      t.d1 = g.m[1];
    }
    if (ctrl >= 0 && c.src(ctrl) == S_SLOT) {  // per-slot control: own op + slot term
      extra.push_back(convert(g, c));
      extra.back().folded = true;
      t.src = S_SLOT;
      t.bit = (uint8_t)c.slot(ctrl);
      t.val = cval;
      run.sterms.push_back(t);
      continue;
    }
    if (!is1(t.d0)) any0 = true;
    t.val = cval;
    if (ctrl < 0) {
      t.src = S_NONE;
      t.bit = 0;
      none.push_back(t);
    } else {
      t.src = c.src(ctrl);
      t.bit = c.bitpos(ctrl);
      (t.src == S_LOCAL ? loc : outer).push_back(t);
    }
  }
  const size_t nterms = loc.size() + outer.size() + none.size();
  if (nterms > 0) {
    if (n_prun >= kMaxPrun || loc.size() > 255 || outer.size() > 255 || none.size() > 255) {
      for (size_t x = i; x < j; ++x) out.push_back(convert(seq[x], c));
      return;
    }
    run.h.flags = any0 ? 1 : 0;
    run.h.nt_local = (uint8_t)loc.size();
    run.h.nt_outer = (uint8_t)outer.size();
    run.h.nt_none = (uint8_t)none.size();
    run.h.wslot = (uint16_t)n_prun++;
    run.terms = loc;
    run.terms.insert(run.terms.end(), outer.begin(), outer.end());
    run.terms.insert(run.terms.end(), none.begin(), none.end());
    out.push_back(run);
  } else {
    for (auto& e : extra) e.folded = false;  // no run to fold them into
  }
  for (auto& e : extra) out.push_back(e);
}

void encode_substage(const std::vector<PGate>& seq, const Ctx& c, int& n_prun,
                     std::vector<FOpIR>& out) {
  size_t i = 0;
  while (i < seq.size()) {
    if (phase_type(seq[i])) {
      uint64_t cands = base_cands(seq[i]);
      size_t j = i + 1;
      while (j < seq.size() && phase_type(seq[j]) && (cands & base_cands(seq[j]))) {
        cands &= base_cands(seq[j]);
        ++j;
      }
      if (j - i >= 2) {
        emit_run(seq, i, j, std::countr_zero(cands), c, n_prun, out);
        i = j;
        continue;
      }
    }
    out.push_back(convert(seq[i], c));
    ++i;
  }
}

}  // namespace

namespace {

// Relabel physical bits a <-> b in a gate (the data of the two bits was swapped).
void swap_bits(PGate& g, int a, int b) {
  auto mv = [&](int p) { return p == a ? b : (p == b ? a : p); };
  g.t0 = mv(g.t0);
  if (pgate_is_two(g)) g.t1 = mv(g.t1);
  for (int j = 0; j < g.nt; ++j) g.tk[j] = mv(g.tk[j]);
  auto mvmask = [&](uint64_t m) {
    const uint64_t ba = (m >> a) & 1ull, bb = (m >> b) & 1ull;
    m &= ~((1ull << a) | (1ull << b));
    return m | (ba << b) | (bb << a);
  };
  g.cmask = mvmask(g.cmask);
  g.cval = mvmask(g.cval);
}

// Bits the next pass's greedy would want in its tile if all k tile bits were
// free (the row bits not reserved): the needed bits of the gates it would take.
uint64_t next_want(const std::vector<PGate>& gates, const std::vector<int>& rem, int k) {
  uint64_t W = 0, blocked = 0;
  for (int gi : rem) {
    const PGate& g = gates[gi];
    const uint64_t all = pgate_bits(g);
    if (all & blocked) {
      blocked |= all;
      continue;
    }
    const uint64_t nw = W | need_mask(g);
    if (popc(nw) <= k) W = nw;
    else blocked |= all;
  }
  return W;
}

struct Group {
  std::vector<PGate> gates;
  uint64_t G = 0;
};

// Non-diagonal gates a pass with tile set T would take from `rem` (in order;
// a gate is taken iff its non-diagonal targets lie in T and no earlier
// deferred gate shares a bit with it).  Stops once every bit of T is blocked.
int score_tile(const std::vector<PGate>& gates, const std::vector<int>& rem, uint64_t T) {
  uint64_t blocked = 0;
  int sc = 0;
  for (int gi : rem) {
    const PGate& g = gates[gi];
    const uint64_t all = pgate_bits(g);
    const uint64_t nd = need_mask(g);
    if (!(all & blocked) && (nd & ~T) == 0) {
      sc += nd != 0;
      continue;
    }
    blocked |= all;
    if ((blocked & T) == T) break;
  }
  return sc;
}

// Tile set for the next pass: in-order greedy growth from `fixed`, then hill
// climbing over single-bit exchanges (bits of `fixed` stay) on score_tile.
uint64_t choose_tile(const std::vector<PGate>& gates, const std::vector<int>& rem, uint64_t fixed, int k, int n,
                     int seeds) {
  uint64_t T = fixed, blocked = 0;
  for (int gi : rem) {
    const PGate& g = gates[gi];
    const uint64_t all = pgate_bits(g);
    if (all & blocked) {
      blocked |= all;
      continue;
    }
    const uint64_t nt = T | need_mask(g);
    if (popc(nt) <= k) T = nt;
    else blocked |= all;
  }
  const uint64_t full = n >= 64 ? ~0ull : (1ull << n) - 1;
  // hill climbing over single-bit additions / exchanges (bits of `fixed` stay)
  auto climb = [&](uint64_t T0, int& sc0) {
    uint64_t Tc = T0;
    int best = score_tile(gates, rem, Tc);
    for (int it = 0; it < 64; ++it) {
      uint64_t bestT = 0;
      const uint64_t outs = full & ~Tc;
      if (popc(Tc) < k) {
        for (uint64_t o = outs; o; o &= o - 1) {
          const uint64_t t2 = Tc | (o & -o);
          const int sc = score_tile(gates, rem, t2);
          if (sc > best) best = sc, bestT = t2;
        }
      } else {
        for (uint64_t i = Tc & ~fixed; i; i &= i - 1)
          for (uint64_t o = outs; o; o &= o - 1) {
            const uint64_t t2 = (Tc & ~(i & -i)) | (o & -o);
            const int sc = score_tile(gates, rem, t2);
            if (sc > best) best = sc, bestT = t2;
          }
      }
      if (!bestT) break;
      Tc = bestT;
    }
    sc0 = best;
    return Tc;
  };
  int best;
  uint64_t bestT = climb(T, best);
  if (seeds) {
    // more starting points: every window of consecutive free bits (1-D
    // brickwork circuits want contiguous qubit ranges), seeds == 1: the best
    // window is climbed; seeds == 2: every window is climbed
    const int free_k = k - popc(fixed);
    uint64_t bw = 0;
    int bws = -1;
    for (int a = 0; a + free_k <= n && free_k > 0; ++a) {
      uint64_t W = fixed;
      int got = 0;
      for (int b = a; b < n && got < free_k; ++b)
        if (!((fixed >> b) & 1ull)) {
          W |= 1ull << b;
          ++got;
        }
      if (got < free_k) break;
      if (seeds >= 2) {
        int sc;
        const uint64_t Tc = climb(W, sc);
        if (sc > best) best = sc, bestT = Tc;
      } else {
        const int sc = score_tile(gates, rem, W);
        if (sc > bws) bws = sc, bw = W;
      }
    }
    if (seeds == 1 && bws >= 0) {
      int sc;
      const uint64_t Tc = climb(bw, sc);
      if (sc > best) best = sc, bestT = Tc;
    }
  }
  return bestT;
}

}  // namespace

namespace {

// Sub-stage groups of one pass: list scheduling over the pass's gates (a
// gate is ready once every earlier gate sharing a bit with it is placed).
// A group first takes, lowest index first, every ready gate whose
// non-diagonal targets already lie in its slot set G; then it grows G by the
// ready gate adding the fewest bits (<= kSlotBits).  Gates keep their
// relative order on every bit, so the product is unchanged; brickwork layers
// fold into triangles of 3-4 blocks per 4-bit group instead of 2.
std::vector<Group> form_groups(const std::vector<PGate>& seq) {
  const int m = (int)seq.size();
  std::vector<std::vector<int>> succ(m);
  std::vector<int> npred(m, 0);
  int last[64];
  for (int b = 0; b < 64; ++b) last[b] = -1;
  for (int j = 0; j < m; ++j) {
    int preds[64], np = 0;
    for (uint64_t x = pgate_bits(seq[j]); x; x &= x - 1) {
      const int b = std::countr_zero(x);
      if (last[b] >= 0 && std::find(preds, preds + np, last[b]) == preds + np) preds[np++] = last[b];
      last[b] = j;
    }
    for (int i = 0; i < np; ++i) succ[preds[i]].push_back(j);
    npred[j] = np;
  }
  std::vector<char> ready(m, 0), done(m, 0);
  for (int j = 0; j < m; ++j) ready[j] = npred[j] == 0;
  std::vector<Group> groups;
  int left = m;
  auto place = [&](Group& gr, int j) {
    gr.G |= need_mask(seq[j]);
    gr.gates.push_back(seq[j]);
    done[j] = 1;
    ready[j] = 0;
    --left;
    for (int s2 : succ[j])
      if (--npred[s2] == 0) ready[s2] = 1;
  };
  while (left > 0) {
    Group gr;
    for (;;) {
      int pick = -1;
      for (int j = 0; j < m && pick < 0; ++j)
        if (ready[j] && (need_mask(seq[j]) & ~gr.G) == 0) pick = j;
      if (pick >= 0) {
        place(gr, pick);
        continue;
      }
      int best = kSlotBits + 1;
      for (int j = 0; j < m; ++j) {
        if (!ready[j]) continue;
        const int c = popc(gr.G | need_mask(seq[j]));
        if (c < best) best = c, pick = j;
      }
      if (pick < 0 || best > kSlotBits) break;
      place(gr, pick);
    }
    groups.push_back(std::move(gr));
  }
  return groups;
}

// Each swap joins the first group at or after the last one touching its bits
// that has slot room; else a new trailing group (order of swaps sharing a bit
// is kept: earlier ones count as touching).
void place_swaps(std::vector<Group>& groups, const std::vector<std::pair<int, int>>& swaps) {
  for (auto [a, b] : swaps) {
    const uint64_t ab = (1ull << a) | (1ull << b);
    size_t j = 0;
    for (size_t x = 0; x < groups.size(); ++x)
      for (const PGate& g : groups[x].gates)
        if (pgate_bits(g) & ab) j = x;
    PGate sw;
    sw.kind = GK::SWAP2;
    sw.t0 = std::max(a, b);
    sw.t1 = std::min(a, b);
    size_t x = j;
    while (x < groups.size() && popc(groups[x].G | ab) > kSlotBits) ++x;
    if (x == groups.size()) groups.emplace_back();
    groups[x].G |= ab;
    groups[x].gates.push_back(sw);
  }
}

// Encode one pass over tile set T from its sub-stage groups.
void emit_pass(int n, int k, int rb, uint64_t T, const std::vector<Group>& groups, FusedPlan& plan) {
  FusedPassPlan pp{};
  const Frame f = make_frame(n, rb, T);
  PassDesc& d = pp.desc;
  d.k = k;
  d.rb = rb;
  d.pshift = rb;
  d.g4 = 0;
  d.rank_bits = 0;
  d.addr_bits = 0;
  d.tile0 = 0;
  d.addr_strip = 0;
  d.grp = 0;
  d.pad1_ = 0;
  for (int h = 0; h < 8; ++h) d.sub_addr[h] = d.sub_state[h] = 0;
  d.n_hi = 0;
  for (int p = rb; p < n; ++p)
    if (T & (1ull << p)) d.hi_pos[d.n_hi++] = p;
  d.n_outer = 0;
  for (int p = 0; p < n; ++p)
    if (!(T & (1ull << p))) d.outer_pos[d.n_outer++] = p;
  d.n_tiles = 1ull << (n - k);
  int n_prun = 0;
  for (const Group& gr : groups) {
    const uint64_t G = gr.G;
    // pad G with the highest tile-local bits (lanes then walk contiguous rows)
    bool in_g[64] = {false};
    for (int p = 0; p < n; ++p)
      if (G & (1ull << p)) in_g[f.local_of[p]] = true;
    int cnt = popc(G);
    for (int l = f.n_local - 1; l >= 0 && cnt < kSlotBits; --l) {
      if (in_g[l]) continue;
      in_g[l] = true;
      ++cnt;
    }
    SubStageDesc sd{};
    Ctx c;
    c.f = &f;
    for (int l = 0; l < 64; ++l) c.slot_of_local[l] = -1;
    int j = 0;
    for (int l = 0; l < f.n_local; ++l)
      if (in_g[l]) {
        sd.g[j] = l;
        c.slot_of_local[l] = j++;
      }
    sd.op_begin = (int)pp.ops.size();
    encode_substage(gr.gates, c, n_prun, pp.ops);
    sd.op_end = (int)pp.ops.size();
    if (sd.op_end > sd.op_begin) pp.subs.push_back(sd);
  }
  d.n_prun = (uint32_t)n_prun;
  factor_pass_scalars(pp);
  if (!pp.subs.empty()) plan.passes.push_back(std::move(pp));
}

// Swaps (applied in order) that move the data of every physical bit back
// home: perm[p] = where the data of home p currently is.
std::vector<std::pair<int, int>> restore_swaps(std::vector<int> cur) {
  std::vector<std::pair<int, int>> out;
  const int n = (int)cur.size();
  std::vector<int> home_at(n);  // home_at[pos] = home whose data is at pos
  for (int h = 0; h < n; ++h) home_at[cur[h]] = h;
  for (int p = 0; p < n; ++p) {
    if (cur[p] == p) continue;
    const int q = cur[p], h = home_at[p];  // p's data at q; position p holds h's data
    out.push_back({p, q});
    cur[p] = p;
    home_at[p] = p;
    cur[h] = q;
    home_at[q] = h;
  }
  return out;
}

// End-of-pass permutation of the tile's bits (remap).  Row positions get
// items (the data of a home bit) the next pass wants, preferring items whose
// home is that row; the other tile positions send items home where possible;
// everything else stays.  Returned as swaps applied in order.
std::vector<std::pair<int, int>> remap_swaps(const std::vector<int>& perm, uint64_t T, uint64_t rows, uint64_t W,
                                             int n) {
  std::vector<int> home_at(n);
  for (int h = 0; h < n; ++h) home_at[perm[h]] = h;
  std::vector<int> want(n, -1);  // target position -> item (home index)
  std::vector<char> placed(n, 0);
  auto in = [](uint64_t m, int p) { return (m >> p) & 1ull; };
  if (W) {  // W == 0: plain restore, rows are ordinary tile positions
    // rows: wanted items whose home is the row, then wanted items already in a row, then others
    for (int r = 0; r < n; ++r)
      if (in(rows, r) && in(T, perm[r]) && in(W, perm[r])) {
        want[r] = r;
        placed[r] = 1;
      }
    for (int r = 0; r < n; ++r)
      if (in(rows, r) && want[r] < 0) {
        const int it = home_at[r];
        if (!placed[it] && in(W, r)) want[r] = it, placed[it] = 1;
      }
    for (int r = 0; r < n; ++r) {
      if (!in(rows, r) || want[r] >= 0) continue;
      for (int p = 0; p < n; ++p) {
        const int it = home_at[p];
        if (in(T, p) && !in(rows, p) && in(W, p) && !placed[it]) {
          want[r] = it, placed[it] = 1;
          break;
        }
      }
    }
    for (int r = 0; r < n; ++r)  // unwanted rows: keep the occupant if free
      if (in(rows, r) && want[r] < 0 && !placed[home_at[r]]) want[r] = home_at[r], placed[home_at[r]] = 1;
  }
  // other tile positions: items going home, then occupants staying
  for (int p = 0; p < n; ++p)
    if (in(T, p) && (!W || !in(rows, p)) && want[p] < 0 && in(T, perm[p]) && !placed[p]) want[p] = p, placed[p] = 1;
  for (int p = 0; p < n; ++p)
    if (in(T, p) && want[p] < 0 && !placed[home_at[p]]) want[p] = home_at[p], placed[home_at[p]] = 1;
  for (int p = 0; p < n; ++p) {
    if (!in(T, p) || want[p] >= 0) continue;
    for (int q = 0; q < n; ++q)
      if (in(T, q) && !placed[home_at[q]]) {
        want[p] = home_at[q], placed[home_at[q]] = 1;
        break;
      }
  }
  // decompose: position p must receive item want[p] (currently at pos[want[p]])
  std::vector<int> pos(perm);
  std::vector<std::pair<int, int>> out;
  for (int p = 0; p < n; ++p) {
    if (!in(T, p) || want[p] < 0) continue;
    const int q = pos[want[p]];
    if (q == p) continue;
    const int other = home_at[p];
    out.push_back({p, q});
    pos[want[p]] = p;
    home_at[p] = want[p];
    pos[other] = q;
    home_at[q] = other;
  }
  return out;
}

}  // namespace

FusedPlan plan_fused(int n, int k, int rb, const std::vector<PGate>& gates_in, bool remap, double flops_budget,
                     int seeds) {
  if (seeds < 0) seeds = getenv("QC_PLAN_SEEDS") ? atoi(getenv("QC_PLAN_SEEDS")) : 0;
  FusedPlan plan;
  std::vector<PGate> gates = gates_in;  // bits relabelled by in-pass remap swaps
  plan.perm.resize(n);
  for (int p = 0; p < n; ++p) plan.perm[p] = p;
  const uint64_t rows = (1ull << rb) - 1;
  std::vector<int> remaining(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) remaining[i] = (int)i;

  while (!remaining.empty()) {
    // search: the tile set is fixed before the take scan (row bits always in it)
    const uint64_t Tc = (remap && n > k) ? choose_tile(gates, remaining, rows, k, n, seeds) : ~0ull;
    uint64_t T = rows;
    uint64_t blocked = 0;
    size_t bytes = 0;
    double flops = 0;  // FP64 budget: past the HBM/FP64 ridge a pass is ALU-bound, and the
                       // gates it still takes cost more time than the next pass's round trip
    std::vector<int> taken, deferred;
    for (int gi : remaining) {
      const PGate& g = gates[gi];
      if (popc(need_mask(g)) + rb > k && n > k) {
        plan.ok = false;
        return plan;
      }
      const uint64_t all = pgate_bits(g);
      if ((all & blocked) || (need_mask(g) & ~Tc)) {
        blocked |= all;
        deferred.push_back(gi);
        continue;
      }
      const uint64_t nt = T | need_mask(g);
      const size_t est = blob_estimate(g);
      const double gf = gate_flops(g);
      if (popc(nt) <= k && bytes + est <= kBlobMax - 4096 &&
          (flops_budget <= 0 || taken.empty() || flops + gf <= flops_budget)) {
        T = nt;
        bytes += est;
        flops += gf;
        taken.push_back(gi);
      } else {
        blocked |= all;
        deferred.push_back(gi);
      }
    }
    if (taken.empty()) {
      plan.ok = false;
      return plan;
    }
    // Remap (n > k): the row bits are in every tile, so whichever qubits sit
    // there ride along in every pass.  Swap row bits the next pass does not
    // want with tile bits it does want -- a permutation of this tile's bits,
    // appended after this pass's last gate on those bits (register renaming
    // inside a sub-stage) -- and relabel the deferred gates accordingly.
    std::vector<std::pair<int, int>> swaps;
    uint64_t W = 0;
    if (remap && n > k && !deferred.empty()) W = choose_tile(gates, deferred, 0, k, n, seeds);
    // last pass: bring every displaced bit home (same layout in and out, so a
    // repeated circuit reuses its plan, JIT kernels and CUDA graph)
    uint64_t D = 0;  // displaced positions (padding with them lets items go home)
    if (remap)
      for (int p = 0; p < n; ++p)
        if (plan.perm[p] != p) D |= 1ull << p;
    for (int p = rb; popc(T) < k && p < n; ++p)  // pad: displaced / wanted bits first
      if ((D | W) & (1ull << p)) T |= 1ull << p;
    for (int p = rb; popc(T) < k && p < n; ++p) T |= 1ull << p;
    if (deferred.empty() && D && (D & ~T) == 0) swaps = restore_swaps(plan.perm);
    else if (W || (deferred.empty() && D)) swaps = remap_swaps(plan.perm, T, rows, W, n);
    std::vector<PGate> seq;
    seq.reserve(taken.size());
    for (int gi : taken) seq.push_back(gates[gi]);
    std::vector<Group> groups = form_groups(seq);
    place_swaps(groups, swaps);
    emit_pass(n, k, rb, T, groups, plan);
    for (auto [a, b] : swaps) {
      for (int gi : deferred) swap_bits(gates[gi], a, b);
      for (int p = 0; p < n; ++p)
        plan.perm[p] = plan.perm[p] == a ? b : (plan.perm[p] == b ? a : plan.perm[p]);
    }
    plan.remap_swaps += (int64_t)swaps.size();
    remaining.swap(deferred);
  }
  // displaced bits the last tile did not hold: swap-only passes.  Item moves
  // (position -> home) form cycles; a tile fixes every move whose two ends it
  // holds, so each pass grows T from the row bits by the position closing
  // the most moves.
  if (getenv("QC_PLAN_DEBUG")) {
    int nd = 0;
    for (int p = 0; p < n; ++p) nd += plan.perm[p] != p;
    fprintf(stderr, "plan: %zu passes, %d displaced bits\n", plan.passes.size(), nd);
  }
  for (int guard = 0; guard < 64; ++guard) {
    std::vector<int> home_at(n);
    for (int h = 0; h < n; ++h) home_at[plan.perm[h]] = h;
    uint64_t D = 0;
    for (int p = 0; p < n; ++p)
      if (plan.perm[p] != p) D |= 1ull << p;
    if (!D) break;
    uint64_t T = rows;
    auto edges = [&](uint64_t t) {  // moves with both ends in t
      int e = 0;
      for (int p = 0; p < n; ++p)
        if (((D >> p) & 1) && ((t >> p) & 1) && ((t >> home_at[p]) & 1)) ++e;
      return e;
    };
    while (popc(T) < k && (D & ~T)) {
      int bestp = -1, beste = -1;
      for (uint64_t o = D & ~T; o; o &= o - 1) {
        const int p = std::countr_zero(o);
        const int e = edges(T | (1ull << p));
        if (e > beste) beste = e, bestp = p;
      }
      T |= 1ull << bestp;
    }
    for (int p = rb; popc(T) < k && p < n; ++p) T |= 1ull << p;
    const std::vector<std::pair<int, int>> chunk = remap_swaps(plan.perm, T, rows, 0, n);
    if (chunk.empty()) break;
    std::vector<Group> groups;
    place_swaps(groups, chunk);
    emit_pass(n, k, rb, T, groups, plan);
    for (auto [a, b] : chunk)
      for (int p = 0; p < n; ++p)
        plan.perm[p] = plan.perm[p] == a ? b : (plan.perm[p] == b ? a : plan.perm[p]);
    plan.remap_swaps += (int64_t)chunk.size();
    ++plan.restore_passes;
  }
  for (int p = 0; p < n; ++p)
    if (plan.perm[p] != p) plan.ok = false;  // (cannot happen: every pass fixes >= 1 move)
  if (getenv("QC_PLAN_DEBUG"))
    for (size_t i = 0; i < plan.passes.size(); ++i) {
      const PassDesc& d = plan.passes[i].desc;
      uint64_t T = (1ull << d.rb) - 1;
      for (int j = 0; j < d.n_hi; ++j) T |= 1ull << d.hi_pos[j];
      const int runs = popc(T & ~(T << 1));  // runs of consecutive tile bits (TMA box dims)
      fprintf(stderr, "pass %zu: subs %zu ops %zu flops/amp %.1f runs %d\n", i, plan.passes[i].subs.size(),
              plan.passes[i].ops.size(), pass_flops_per_amp(plan.passes[i]), runs);
    }
  return plan;
}

// Algorithmic flops per state amplitude of a fused plan: what the fused ops
// must compute, counted as complex arithmetic (a general complex multiply 6
// flops, multiply-accumulate 8; multiplying by +-1 / +-i free, accumulating
// it 2), times the fraction of amplitudes each op touches (predicates halve
// it per bit, identity rows and the d0 = 1 half of a diagonal are skipped).
// The ALU roofline of bench.py divides this work by the pass time.
double pass_flops_per_amp(const FusedPassPlan& pp) {
  auto unit = [](cd z) {
    return (std::abs(z.imag()) == 0.0 && std::abs(z.real()) == 1.0) ||
           (z.real() == 0.0 && std::abs(z.imag()) == 1.0);
  };
  double total = 0;
  {
    for (const auto& o : pp.ops) {
      if (o.folded) continue;
      const FHdr& h = o.h;
      const double pred = std::ldexp(1.0, -(popc(h.smask) + popc(h.lmask) + popc(h.omask)));
      if (h.kind == F_M1 || h.kind == F_M2) {
        const int dim = h.kind == F_M1 ? 2 : 4;
        double f = 0;
        for (int r = 0; r < dim; ++r) {
          double fr = 0;
          bool first = true, ident = true;
          for (int c = 0; c < dim; ++c) {
            const cd z = o.dense[r * dim + c];
            if (r == c ? !(z.real() == 1.0 && z.imag() == 0.0) : !is0(z)) ident = false;
            if (is0(z)) continue;
            fr += first ? (unit(z) ? 0 : 6) : (unit(z) ? 2 : 8);
            first = false;
          }
          if (!ident) f += fr;
        }
        total += f / dim * pred;
      } else if (h.kind == F_MK) {
        const int dim = 1 << h.sb1;
        double f = 0;
        for (int r = 0; r < dim; ++r) {
          bool first = true;
          for (int cc = 0; cc < dim; ++cc) {
            const cd z = o.mk[(size_t)r * dim + cc];
            if (is0(z)) continue;
            f += first ? (unit(z) ? 0 : 6) : (unit(z) ? 2 : 8);
            first = false;
          }
        }
        total += f / dim * pred;
      } else if (h.kind == F_DSCALE) {
        total += 6.0 * ((h.flags & 1) ? 0.5 : 1.0) * pred;
      } else {  // F_PRUN: one complex factor per amplitude (the d0 = 1 half skipped)
        total += 6.0 * ((h.flags & 1) || !o.sterms.empty() ? 1.0 : 0.5) * pred;
      }
    }
  }
  return total;
}

double plan_flops_per_amp(const FusedPlan& plan) {
  double total = 0;
  for (const auto& pp : plan.passes) total += pass_flops_per_amp(pp);
  return total;
}

namespace {
size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <typename T>
void pack_pass(FusedPassPlan& pp, std::vector<uint8_t>& blob) {
  using CT2 = T[2];
  size_t ncoef = 0, nterm = 0;
  for (auto& o : pp.ops) {
    ncoef += o.coefs.size();
    nterm += o.terms.size();
  }
  PassDesc& d = pp.desc;
  d.n_sub = (uint32_t)pp.subs.size();
  d.n_ops = (uint32_t)pp.ops.size();
  const size_t off_hdr = align16(pp.subs.size() * sizeof(SubStageDesc));
  const size_t off_coef = align16(off_hdr + pp.ops.size() * sizeof(FHdr));
  const size_t off_term = align16(off_coef + ncoef * sizeof(CT2));
  const size_t total = align16(off_term + nterm * sizeof(FTermT<T>));
  d.off_hdr = (uint32_t)off_hdr;
  d.off_coef = (uint32_t)off_coef;
  d.off_term = (uint32_t)off_term;
  d.blob_bytes = (uint32_t)total;
  d.blob_off = blob.size();
  blob.resize(blob.size() + total, 0);
  uint8_t* base = blob.data() + d.blob_off;
  std::memcpy(base, pp.subs.data(), pp.subs.size() * sizeof(SubStageDesc));
  size_t ci = 0, ti = 0;
  for (size_t i = 0; i < pp.ops.size(); ++i) {
    FOpIR& o = pp.ops[i];
    FHdr h = o.h;
    if (h.kind == F_PRUN) {
      h.coef = (uint32_t)ti;
      for (auto& t : o.terms) {
        FTermT<T> ft{};
        ft.src = t.src;
        ft.bit = t.bit;
        ft.val = t.val;
        ft.d0one = is1(t.d0) ? 1 : 0;
        ft.d0r = (T)t.d0.real();
        ft.d0i = (T)t.d0.imag();
        ft.d1r = (T)t.d1.real();
        ft.d1i = (T)t.d1.imag();
        std::memcpy(base + off_term + ti * sizeof(FTermT<T>), &ft, sizeof ft);
        ++ti;
      }
    } else {
      h.coef = (uint32_t)ci;
      for (auto& z : o.coefs) {
        T v[2] = {(T)z.real(), (T)z.imag()};
        std::memcpy(base + off_coef + ci * sizeof(CT2), v, sizeof v);
        ++ci;
      }
    }
    std::memcpy(base + off_hdr + i * sizeof(FHdr), &h, sizeof h);
  }
}
}  // namespace

std::vector<uint8_t> pack_plan(FusedPlan& plan, bool dbl) {
  std::vector<uint8_t> blob;
  for (auto& pp : plan.passes) {
    if (dbl)
      pack_pass<double>(pp, blob);
    else
      pack_pass<float>(pp, blob);
  }
  return blob;
}

// Exported for dist.cu (pair segments relabel a rank bit into plan bit n_loc).
void pgate_swap_bits(PGate& g, int a, int b) { swap_bits(g, a, b); }

}  // namespace qc
