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
#include <cstring>

#include "qc_internal.h"

namespace qc {
namespace {

inline int popc(uint64_t x) { return std::popcount(x); }

uint64_t target_mask(const PGate& g) {
  uint64_t m = 1ull << g.t0;
  if (pgate_is_two(g)) m |= 1ull << g.t1;
  return m;
}
uint64_t need_mask(const PGate& g) { return g.kind == GK::DIAG1 ? 0ull : target_mask(g); }

size_t blob_estimate(const PGate& g) {
  if (g.kind == GK::DIAG1) return 48;
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

// A single (non-run) gate -> one fused op.
FOpIR convert(const PGate& g, const Ctx& c) {
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

FusedPlan plan_fused(int n, int k, int rb, const std::vector<PGate>& gates) {
  FusedPlan plan;
  std::vector<int> remaining(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) remaining[i] = (int)i;

  while (!remaining.empty()) {
    uint64_t T = (1ull << rb) - 1;
    uint64_t blocked = 0;
    size_t bytes = 0;
    std::vector<int> taken, deferred;
    for (int gi : remaining) {
      const PGate& g = gates[gi];
      if (popc(need_mask(g)) + rb > k && n > k) {
        plan.ok = false;
        return plan;
      }
      const uint64_t all = pgate_bits(g);
      if (all & blocked) {
        blocked |= all;
        deferred.push_back(gi);
        continue;
      }
      const uint64_t nt = T | need_mask(g);
      const size_t est = blob_estimate(g);
      if (popc(nt) <= k && bytes + est <= kBlobMax - 4096) {
        T = nt;
        bytes += est;
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
    for (int p = rb; popc(T) < k && p < n; ++p) T |= 1ull << p;

    FusedPassPlan pp{};
    const Frame f = make_frame(n, rb, T);
    PassDesc& d = pp.desc;
    d.k = k;
    d.rb = rb;
    d.pshift = rb;
    d.g4 = 0;
    d.rank_bits = 0;
    d.addr_bits = 0;
    d.n_hi = 0;
    for (int p = rb; p < n; ++p)
      if (T & (1ull << p)) d.hi_pos[d.n_hi++] = p;
    d.n_outer = 0;
    for (int p = 0; p < n; ++p)
      if (!(T & (1ull << p))) d.outer_pos[d.n_outer++] = p;
    d.n_tiles = 1ull << (n - k);
    int n_prun = 0;

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
      std::vector<PGate> seq;
      for (size_t x = gi; x < gj; ++x) seq.push_back(gates[taken[x]]);
      sd.op_begin = (int)pp.ops.size();
      encode_substage(seq, c, n_prun, pp.ops);
      sd.op_end = (int)pp.ops.size();
      if (sd.op_end > sd.op_begin) pp.subs.push_back(sd);
      gi = gj;
    }
    d.n_prun = (uint32_t)n_prun;
    factor_pass_scalars(pp);
    if (!pp.subs.empty()) plan.passes.push_back(std::move(pp));
    remaining.swap(deferred);
  }
  return plan;
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

}  // namespace qc
