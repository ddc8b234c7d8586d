// fuse.cpp -- gate-block fusion (host): merge consecutive gates acting on the
// same <= 2 physical bits into one block, then classify the block's exact
// structure (identity / diagonal / permutation / 2-sparse / dense).
//
// Why: on B200 a complex128 fused pass is bounded by the FP64 pipe, not HBM,
// once a tile holds more than ~10 dense 1q gates (DESIGN "FP64 ridge").
// Merging gates that act on the same qubit pair multiplies their matrices on
// the host, so e.g. a TFXY pair block  RZ RZ . CNOT . RX (x) RZ . CNOT . RZ RZ
// (8 gates, ~28 FP64 instr/amplitude) becomes ONE 4x4 whose rows have two
// non-zeros (exactly: zeros stay exact zeros under multiplication), costing 8
// FP64 instr/amplitude.  The product of the blocks is the product of the gates
// (eq:kron composed in order): a block only absorbs gates/blocks
// that are the latest on all of their bits, so every reordering is a
// commutation of operators on disjoint bits.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>

#include "qc_internal.h"

namespace qc {

bool pgate_is_two(const PGate& g) {
  return g.kind == GK::DENSE2 || g.kind == GK::SWAP2 || g.kind == GK::SPARSE2 ||
         g.kind == GK::PERM2 || g.kind == GK::DIAG2;
}

uint64_t pgate_targets(const PGate& g) {
  if (g.kind == GK::DENSEK) {
    uint64_t m = 0;
    for (int j = 0; j < g.nt; ++j) m |= 1ull << g.tk[j];
    return m;
  }
  uint64_t m = 1ull << g.t0;
  if (pgate_is_two(g)) m |= 1ull << g.t1;
  return m;
}

uint64_t pgate_bits(const PGate& g) { return g.cmask | pgate_targets(g); }

void pgate_dense4(const PGate& g, cd out[16]) {
  for (int i = 0; i < 16; ++i) out[i] = 0;
  switch (g.kind) {
    case GK::DENSE2: for (int i = 0; i < 16; ++i) out[i] = g.m[i]; break;
    case GK::SWAP2: out[0] = 1; out[6] = 1; out[9] = 1; out[15] = 1; break;
    case GK::SPARSE2:
      for (int r = 0; r < 4; ++r) {
        out[4 * r + g.col[2 * r]] += g.m[2 * r];
        out[4 * r + g.col[2 * r + 1]] += g.m[2 * r + 1];
      }
      break;
    case GK::PERM2: for (int r = 0; r < 4; ++r) out[4 * r + g.col[r]] = 1; break;
    case GK::DIAG2: for (int r = 0; r < 4; ++r) out[5 * r] = g.m[r]; break;
    default: break;
  }
}

namespace {

uint64_t gate_bits(const PGate& g) { return pgate_bits(g); }

// Apply g to a small vector over the physical bits `bits` (bits[0] = MSB of
// the local index).  Every bit g touches must be in `bits`.
void apply_small(const PGate& g, const int* bits, int nb, cd* v) {
  const int dim = 1 << nb;
  auto lpos = [&](int p) {
    for (int i = 0; i < nb; ++i)
      if (bits[i] == p) return nb - 1 - i;
    return -1;
  };
  uint32_t cm = 0, cv = 0;
  for (int p = 0; p < 64; ++p)
    if (g.cmask & (1ull << p)) {
      cm |= 1u << lpos(p);
      if (g.cval & (1ull << p)) cv |= 1u << lpos(p);
    }
  const uint32_t b0 = 1u << lpos(g.t0);
  const bool two = pgate_is_two(g);
  const uint32_t b1 = two ? (1u << lpos(g.t1)) : 0u;
  std::vector<cd> out(v, v + dim);
  for (int l = 0; l < dim; ++l) {
    if ((l & b0) || (l & b1) || ((uint32_t)l & cm) != cv) continue;
    if (!two) {
      const cd a = v[l], b = v[l | b0];
      switch (g.kind) {
        case GK::DENSE1:
          out[l] = g.m[0] * a + g.m[1] * b;
          out[l | b0] = g.m[2] * a + g.m[3] * b;
          break;
        case GK::PERM1:
          out[l] = b;
          out[l | b0] = a;
          break;
        default:  // DIAG1
          out[l] = g.m[0] * a;
          out[l | b0] = g.m[1] * b;
          break;
      }
    } else {
      const uint32_t id[4] = {(uint32_t)l, l | b1, l | b0, l | b0 | b1};  // index 2*bit(t0)+bit(t1)
      cd x[4];
      for (int r = 0; r < 4; ++r) x[r] = v[id[r]];
      for (int r = 0; r < 4; ++r) {
        cd acc = 0;
        switch (g.kind) {
          case GK::DENSE2:
            for (int c = 0; c < 4; ++c) acc += g.m[4 * r + c] * x[c];
            break;
          case GK::SWAP2: acc = x[r == 1 ? 2 : (r == 2 ? 1 : r)]; break;
          case GK::SPARSE2: acc = g.m[2 * r] * x[g.col[2 * r]] + g.m[2 * r + 1] * x[g.col[2 * r + 1]]; break;
          case GK::PERM2: acc = x[g.col[r]]; break;
          default: acc = g.m[r] * x[r]; break;  // DIAG2
        }
        out[id[r]] = acc;
      }
    }
  }
  std::copy(out.begin(), out.end(), v);
}

struct Block {
  bool alive = true;
  bool raw = false;       // unfusable gate (> 2 bits), kept as is
  uint64_t bits = 0;
  int nb = 0;
  int b[2] = {-1, -1};    // b[0] = higher physical bit (matrix MSB)
  cd M[16];               // dim x dim, row-major
  PGate g;                // raw gate or classified result
  double cost = 0;
};

double gate_cost(const PGate& g) {
  const double ctrl = std::ldexp(1.0, -std::popcount(g.cmask));
  switch (g.kind) {
    case GK::DENSE1: return 8 * ctrl + 1;
    case GK::PERM1: return 0.25 * ctrl + 1;
    case GK::DIAG1: return (g.d0_is_one ? 2 : 4) * ctrl + 1;
    case GK::DENSE2: return 16 + 1;
    case GK::SPARSE2: return 8 + 1;
    case GK::PERM2: case GK::SWAP2: return 0.25 + 1;
    case GK::DIAG2: return 4 + 1;
  }
  return 1;
}

bool is0(cd z) { return z.real() == 0.0 && z.imag() == 0.0; }
bool is1(cd z) { return z.real() == 1.0 && z.imag() == 0.0; }

// Classify an exact matrix on (b[0], b[1]) into the cheapest kernel class.
// Returns false for the identity (block can be dropped).
bool classify(Block& B) {
  const int dim = 1 << B.nb;
  bool ident = true;
  for (int r = 0; r < dim; ++r)
    for (int c = 0; c < dim; ++c)
      if (r == c ? !is1(B.M[r * dim + c]) : !is0(B.M[r * dim + c])) ident = false;
  if (ident) return false;
  PGate& g = B.g;
  g = PGate{};
  g.t0 = B.b[0];
  if (B.nb == 1) {
    const cd* M = B.M;
    if (is0(M[1]) && is0(M[2])) {
      g.kind = GK::DIAG1;
      g.m[0] = M[0];
      g.m[1] = M[3];
      g.d0_is_one = is1(M[0]);
    } else if (is0(M[0]) && is0(M[3]) && is1(M[1]) && is1(M[2])) {
      g.kind = GK::PERM1;
    } else {
      g.kind = GK::DENSE1;
      for (int i = 0; i < 4; ++i) g.m[i] = M[i];
    }
    B.cost = gate_cost(g);
    return true;
  }
  g.t1 = B.b[1];
  const cd* M = B.M;
  int nnz[4] = {0, 0, 0, 0};
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) nnz[r] += !is0(M[4 * r + c]);
  bool diag = true, perm = true;
  for (int r = 0; r < 4; ++r) {
    for (int c = 0; c < 4; ++c) {
      if (r != c && !is0(M[4 * r + c])) diag = false;
      if (!is0(M[4 * r + c]) && !is1(M[4 * r + c])) perm = false;
    }
    if (nnz[r] != 1) perm = false;
  }
  if (diag) {
    int non1 = 0, at = -1;
    for (int r = 0; r < 4; ++r)
      if (!is1(M[5 * r])) { ++non1; at = r; }
    if (non1 == 1) {
      // one phase on |h l> = |at>: DIAG1 on the low bit controlled by the high bit
      g.kind = GK::DIAG1;
      g.t0 = B.b[1];
      g.t1 = -1;
      g.cmask = 1ull << B.b[0];
      g.cval = (uint64_t)((at >> 1) & 1) << B.b[0];
      const int lb = at & 1;
      g.m[0] = lb ? cd(1, 0) : M[5 * at];
      g.m[1] = lb ? M[5 * at] : cd(1, 0);
      g.d0_is_one = lb == 1;
    } else {
      g.kind = GK::DIAG2;
      for (int r = 0; r < 4; ++r) g.m[r] = M[5 * r];
    }
  } else if (perm) {
    g.kind = GK::PERM2;
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c)
        if (is1(M[4 * r + c])) g.col[r] = (int8_t)c;
  } else if (nnz[0] <= 2 && nnz[1] <= 2 && nnz[2] <= 2 && nnz[3] <= 2) {
    g.kind = GK::SPARSE2;
    for (int r = 0; r < 4; ++r) {
      int k = 0;
      int cols[2] = {r, r};
      for (int c = 0; c < 4; ++c)
        if (!is0(M[4 * r + c])) cols[k++] = c;
      if (k == 1) cols[1] = (cols[0] == r) ? (r ^ 1) : r;  // second term has coefficient 0
      g.col[2 * r] = (int8_t)cols[0];
      g.col[2 * r + 1] = (int8_t)cols[1];
      g.m[2 * r] = M[4 * r + cols[0]];
      g.m[2 * r + 1] = M[4 * r + cols[1]];
    }
  } else {
    g.kind = GK::DENSE2;
    for (int i = 0; i < 16; ++i) g.m[i] = M[i];
  }
  B.cost = gate_cost(g);
  return true;
}

void block_matrix_of_gate(const PGate& g, Block& B) {
  const int dim = 1 << B.nb;
  for (int c = 0; c < dim; ++c) {
    cd v[4] = {0, 0, 0, 0};
    v[c] = 1;
    apply_small(g, B.b, B.nb, v);
    for (int r = 0; r < dim; ++r) B.M[r * dim + c] = v[r];
  }
}

// Embed block A (1 or 2 bits, subset of B's bits) into B's bit order.
void embed(const Block& A, const Block& B, cd* out) {
  const int dim = 1 << B.nb;
  for (int c = 0; c < dim; ++c) {
    cd v[4] = {0, 0, 0, 0};
    v[c] = 1;
    // apply A as a dense gate on its own bits
    PGate g;
    if (A.nb == 1) {
      g.kind = GK::DENSE1;
      g.t0 = A.b[0];
      for (int i = 0; i < 4; ++i) g.m[i] = A.M[i];
    } else {
      g.kind = GK::DENSE2;
      g.t0 = A.b[0];
      g.t1 = A.b[1];
      for (int i = 0; i < 16; ++i) g.m[i] = A.M[i];
    }
    apply_small(g, B.b, B.nb, v);
    for (int r = 0; r < dim; ++r) out[r * dim + c] = v[r];
  }
}

void setup_bits(Block& B, uint64_t bits) {
  B.bits = bits;
  B.nb = std::popcount(bits);
  int k = 0;
  for (int p = 63; p >= 0; --p)
    if (bits & (1ull << p)) B.b[k++] = p;
}

}  // namespace

std::vector<PGate> fuse_blocks(const std::vector<PGate>& in, uint64_t local_mask) {
  std::vector<Block> blocks;
  blocks.reserve(in.size());
  int last[64];
  for (int p = 0; p < 64; ++p) last[p] = -1;

  for (const PGate& g : in) {
    const uint64_t Q = gate_bits(g);
    // candidate blocks: the latest item on each of g's bits
    int cand[3];
    int nc = 0;
    bool ok = std::popcount(Q) <= 2 && !(Q & ~local_mask);
    for (int p = 0; p < 64 && ok; ++p) {
      if (!(Q & (1ull << p)) || last[p] < 0) continue;
      const int bi = last[p];
      bool dup = false;
      for (int i = 0; i < nc; ++i) dup |= cand[i] == bi;
      if (dup) continue;
      const Block& B = blocks[bi];
      if (B.raw) { ok = false; break; }
      for (int q = 0; q < 64; ++q)  // B must still be the latest on all its bits
        if ((B.bits & (1ull << q)) && last[q] != bi) ok = false;
      cand[nc++] = bi;
    }
    uint64_t U = Q;
    for (int i = 0; ok && i < nc; ++i) U |= blocks[cand[i]].bits;
    if (ok && std::popcount(U) > 2) ok = false;

    Block NB;
    if (std::popcount(Q) > 2 || (Q & ~local_mask)) {  // > 2 bits, or touches a rank bit: keep as is
      NB.raw = true;
      NB.bits = Q;
      NB.g = g;
      NB.cost = gate_cost(g);
    } else {
      // g alone, on its own bits
      Block G1;
      setup_bits(G1, Q);
      block_matrix_of_gate(g, G1);
      const double g_cost = gate_cost(g);
      bool merged = false;
      if (ok && nc > 0) {
        Block M;
        setup_bits(M, U);
        const int dim = 1 << M.nb;
        // P = product of candidate blocks (disjoint bits -> they commute)
        cd P[16], T[16], E[16];
        for (int i = 0; i < dim * dim; ++i) P[i] = (i % (dim + 1) == 0) ? cd(1, 0) : cd(0, 0);
        double parts = g_cost;
        for (int i = 0; i < nc; ++i) {
          embed(blocks[cand[i]], M, E);
          for (int r = 0; r < dim; ++r)
            for (int c = 0; c < dim; ++c) {
              cd acc = 0;
              for (int k = 0; k < dim; ++k) acc += E[r * dim + k] * P[k * dim + c];
              T[r * dim + c] = acc;
            }
          std::copy(T, T + dim * dim, P);
          parts += blocks[cand[i]].cost;
        }
        embed(G1, M, E);
        for (int r = 0; r < dim; ++r)
          for (int c = 0; c < dim; ++c) {
            cd acc = 0;
            for (int k = 0; k < dim; ++k) acc += E[r * dim + k] * P[k * dim + c];
            M.M[r * dim + c] = acc;
          }
        const bool keep = classify(M);
        const double mcost = keep ? M.cost : 0.0;
        if (mcost <= parts + 1e-9) {
          for (int i = 0; i < nc; ++i) blocks[cand[i]].alive = false;
          merged = true;
          if (!keep) {
            // product is exactly the identity: nothing to apply on these bits
            for (int p = 0; p < 64; ++p)
              if (U & (1ull << p)) last[p] = -1;
            continue;
          }
          NB = M;
        }
      }
      if (!merged) {
        NB = G1;
        if (!classify(NB)) {  // the gate itself is exactly the identity
          continue;
        }
      }
    }
    blocks.push_back(NB);
    const int id = (int)blocks.size() - 1;
    for (int p = 0; p < 64; ++p)
      if (NB.bits & (1ull << p)) last[p] = id;
  }
  std::vector<PGate> out;
  out.reserve(blocks.size());
  for (const Block& B : blocks)
    if (B.alive) out.push_back(B.g);
  return out;
}

}  // namespace qc
