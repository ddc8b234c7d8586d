// cpu_omp.cpp -- libqc_omp.so: the paper's CPU implementation (include/qc_omp.h).
//
// qclab++ runs every gate as ONE `#pragma omp parallel for` over the index loop
// of Algorithms 1-3 (CPU listing of fig:Xgate-cpu-vs-gpu), and
// its CPU-vs-GPU experiments time that program.  This file is that
// program: bit masks m_L / m_C / m_R exactly as P:599-613 and P:829-850 define
// them (64-bit, reading R3), the control-state increment of P:870-874, the
// simplified updates of P:617-631 (X, Y, Z), P:852-854 (CNOT) and P:932-938
// (SWAP), and one more mask per extra control for CCX.  2-qubit
// matrices follow eq:kron over the listed qubits (reading R1).  It is a
// separately built baseline -- libqc.so neither loads nor calls it.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/qc_omp.h"

namespace {

thread_local std::string g_err;

qc_status fail(qc_status st, const char* fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

const int kArity[16] = {1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 1, 2, 2, 3};
const int kNctrl[16] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 0, 0, 1, 0, 2};

// ------------------------------------------------------------ index masks
// Zero bits inserted at the (sorted) qubits q[0] < q[1] < ... < q[k-1]: k+1
// masks, mask i holding the loop-counter bits that land between insertion
// points i-1 and i, shifted left by i (P:599-613 for k = 1: m_R, m_L;
// P:829-850 for k = 2: m_R, m_C, m_L; "2 additional bit masks for
// every additional qubit").  Qubit q is index bit n-1-q (Definition 1).
struct Masks {
  int k;
  uint64_t m[4];
  uint64_t at(uint64_t j) const {
    uint64_t a = 0;
    for (int i = 0; i < k + 1; ++i) a += (j & m[i]) << i;
    return a;
  }
};

// n qubits, k sorted inserted qubits (q ascending = index bits descending)
Masks make_masks(int n, const int* q_sorted, int k) {
  Masks M;
  M.k = k;
  // m_R = 2^{n-q_{k-1}-1} - 1; each further mask spans up to the next insertion
  uint64_t below = 0;  // bits already covered (of the loop counter j < 2^{n-k})
  for (int i = 0; i < k; ++i) {
    const int qi = q_sorted[k - 1 - i];                       // from the least significant insertion
    const uint64_t top = (1ull << (n - qi - 1 - i)) - 1;      // counter bits below insertion i
    M.m[i] = top - below;
    below = top;
  }
  M.m[k] = ((1ull << (n - k)) - 1) - below;                   // m_L
  return M;
}

template <typename T>
using cx = std::complex<T>;

template <typename T>
void gate_1q(int n, int q, cx<T>* x, const cx<T> u[4], int op, int nt) {
  const int64_t jmax = (int64_t)1 << (n - 1);
  const int qs[1] = {q};
  const Masks M = make_masks(n, qs, 1);  // Alg. alg:1q lines 1-2
  const uint64_t off = 1ull << (n - q - 1);
  switch (op) {
    case QC_X:  // psi[a] = phi[b], psi[b] = phi[a]
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t a = M.at((uint64_t)j), b = a + off;
        const cx<T> t = x[a];
        x[a] = x[b];
        x[b] = t;
      }
      break;
    case QC_Y:  // psi[a] = -i phi[b], psi[b] = i phi[a]
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t a = M.at((uint64_t)j), b = a + off;
        const cx<T> pa = x[a], pb = x[b];
        x[a] = cx<T>(pb.imag(), -pb.real());
        x[b] = cx<T>(-pa.imag(), pa.real());
      }
      break;
    case QC_Z: case QC_P:  // only the b_j half changes
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t b = M.at((uint64_t)j) + off;
        x[b] = u[3] * x[b];
      }
      break;
    case QC_RZ:  // diagonal
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t a = M.at((uint64_t)j), b = a + off;
        x[a] = u[0] * x[a];
        x[b] = u[3] * x[b];
      }
      break;
    default:  // Alg. alg:1q lines 3-6
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t a = M.at((uint64_t)j), b = a + off;
        const cx<T> pa = x[a], pb = x[b];
        x[a] = u[0] * pa + u[1] * pb;
        x[b] = u[2] * pa + u[3] * pb;
      }
  }
}

// Controlled 1-qubit gate with nc (1 or 2) controls: Alg. alg:ctrl-1q.
template <typename T>
void gate_ctrl_1q(int n, const int* ctrl, int nc, uint32_t cstate, int qt, cx<T>* x, const cx<T> u[4], int op,
                  int nt) {
  int qs[3];
  int k = 0;
  for (int i = 0; i < nc; ++i) qs[k++] = ctrl[i];
  qs[k++] = qt;
  for (int i = 1; i < k; ++i)  // sort ascending (q_0 = min, ...)
    for (int j = i; j > 0 && qs[j] < qs[j - 1]; --j) std::swap(qs[j], qs[j - 1]);
  const Masks M = make_masks(n, qs, k);
  uint64_t cadd = 0;  // one-controlled: a_j, b_j += 2^{n-q_c-1}
  for (int i = 0; i < nc; ++i)
    if ((cstate >> i) & 1u) cadd += 1ull << (n - ctrl[i] - 1);
  const uint64_t off = 1ull << (n - qt - 1);
  const int64_t jmax = (int64_t)1 << (n - k);
  switch (op) {
    case QC_CNOT: case QC_CCX:  // swaps half of the elements
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t a = M.at((uint64_t)j) + cadd, b = a + off;
        const cx<T> t = x[a];
        x[a] = x[b];
        x[b] = t;
      }
      break;
    case QC_CZ: case QC_CP:  // diagonal with u00 = 1: only b_j
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t b = M.at((uint64_t)j) + cadd + off;
        x[b] = u[3] * x[b];
      }
      break;
    default:  // CU1: lines 7-8 of Alg. alg:ctrl-1q
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t j = 0; j < jmax; ++j) {
        const uint64_t a = M.at((uint64_t)j) + cadd, b = a + off;
        const cx<T> pa = x[a], pb = x[b];
        x[a] = u[0] * pa + u[1] * pb;
        x[b] = u[2] * pa + u[3] * pb;
      }
  }
}

// 2-qubit gate on the listed pair (qa, qb): Alg. alg:2q, matrix index
// 2*bit(qa) + bit(qb) (eq:kron, reading R1).
template <typename T>
void gate_2q(int n, int qa, int qb, cx<T>* x, const cx<T> u[16], bool swap, int nt) {
  const int qs[2] = {std::min(qa, qb), std::max(qa, qb)};
  const Masks M = make_masks(n, qs, 2);
  const uint64_t ob = 1ull << (n - qb - 1), oc = 1ull << (n - qa - 1);
  const int64_t jmax = (int64_t)1 << (n - 2);
  if (swap) {  // psi[b] = phi[c], psi[c] = phi[b]
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t j = 0; j < jmax; ++j) {
      const uint64_t a = M.at((uint64_t)j);
      const cx<T> t = x[a + ob];
      x[a + ob] = x[a + oc];
      x[a + oc] = t;
    }
    return;
  }
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t j = 0; j < jmax; ++j) {
    const uint64_t a = M.at((uint64_t)j), id[4] = {a, a + ob, a + oc, a + ob + oc};
    cx<T> p[4];
    for (int c = 0; c < 4; ++c) p[c] = x[id[c]];
    for (int r = 0; r < 4; ++r) x[id[r]] = u[4 * r] * p[0] + u[4 * r + 1] * p[1] + u[4 * r + 2] * p[2] + u[4 * r + 3] * p[3];
  }
}

template <typename T>
void apply_one(int n, cx<T>* x, const qc_gate& g, int nt) {
  using C = cx<T>;
  const double th = g.theta, c = std::cos(th / 2), s = std::sin(th / 2), h = 1.0 / std::sqrt(2.0);
  const std::complex<double> I(0, 1);
  std::complex<double> ud[16] = {};
  switch (g.op) {  // DESIGN R4 matrices
    case QC_H: ud[0] = h; ud[1] = h; ud[2] = h; ud[3] = -h; break;
    case QC_Z: case QC_CZ: ud[0] = 1; ud[3] = -1; break;
    case QC_P: case QC_CP: ud[0] = 1; ud[3] = std::exp(I * th); break;
    case QC_RX: ud[0] = c; ud[1] = -I * s; ud[2] = -I * s; ud[3] = c; break;
    case QC_RY: ud[0] = c; ud[1] = -s; ud[2] = s; ud[3] = c; break;
    case QC_RZ: ud[0] = std::exp(-I * (th / 2)); ud[3] = std::exp(I * (th / 2)); break;
    case QC_U1: case QC_CU1:
      for (int i = 0; i < 4; ++i) ud[i] = {g.m[2 * i], g.m[2 * i + 1]};
      break;
    case QC_U2:
      for (int i = 0; i < 16; ++i) ud[i] = {g.m[2 * i], g.m[2 * i + 1]};
      break;
    default: break;
  }
  C u[16];
  for (int i = 0; i < 16; ++i) u[i] = C((T)ud[i].real(), (T)ud[i].imag());
  switch (g.op) {
    case QC_SWAP: gate_2q<T>(n, g.qubits[0], g.qubits[1], x, u, true, nt); break;
    case QC_U2: gate_2q<T>(n, g.qubits[0], g.qubits[1], x, u, false, nt); break;
    case QC_CNOT: case QC_CZ: case QC_CP: case QC_CU1: case QC_CCX: {
      const int nc = kNctrl[g.op];
      gate_ctrl_1q<T>(n, g.qubits, nc, g.ctrl_state, g.qubits[nc], x, u, g.op, nt);
      break;
    }
    default: gate_1q<T>(n, g.qubits[0], x, u, g.op, nt);
  }
}

qc_status validate(int n, const qc_gate& g, size_t i) {
  if (g.op == QC_MGATE) return fail(QC_ERR_UNSUPPORTED, "op %zu: generic gates are not in the paper's CPU program", i);
  if (g.op < 0 || g.op > 15) return fail(QC_ERR_INVALID_ARG, "op %zu: unknown op code %d", i, g.op);
  if (g.flags) return fail(QC_ERR_INVALID_ARG, "op %zu: flags must be 0", i);
  for (int t = 0; t < kArity[g.op]; ++t) {
    if (g.qubits[t] < 0 || g.qubits[t] >= n) return fail(QC_ERR_INVALID_ARG, "op %zu: qubit %d out of range", i, g.qubits[t]);
    for (int u = 0; u < t; ++u)
      if (g.qubits[u] == g.qubits[t]) return fail(QC_ERR_INVALID_ARG, "op %zu: qubit %d repeated", i, g.qubits[t]);
  }
  if (!std::isfinite(g.theta)) return fail(QC_ERR_INVALID_ARG, "op %zu: theta not finite", i);
  for (int e = 0; e < 32; ++e)
    if (!std::isfinite(g.m[e])) return fail(QC_ERR_INVALID_ARG, "op %zu: matrix entry not finite", i);
  return QC_OK;
}

}  // namespace

extern "C" {

qc_status qc_omp_run(int n, qc_precision p, void* x, const qc_gate* ops, size_t n_ops, int nthreads) {
  if (n < 1 || n > 40) return fail(QC_ERR_INVALID_ARG, "n=%d outside [1,40]", n);
  if (p != QC_COMPLEX64 && p != QC_COMPLEX128) return fail(QC_ERR_INVALID_ARG, "bad precision");
  if (!x) return fail(QC_ERR_INVALID_ARG, "state is NULL");
  if (n_ops && !ops) return fail(QC_ERR_INVALID_ARG, "ops is NULL");
  for (size_t i = 0; i < n_ops; ++i) {
    const qc_status st = validate(n, ops[i], i);
    if (st != QC_OK) return st;
  }
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
  for (size_t i = 0; i < n_ops; ++i) {
    if (p == QC_COMPLEX128)
      apply_one<double>(n, reinterpret_cast<cx<double>*>(x), ops[i], nt);
    else
      apply_one<float>(n, reinterpret_cast<cx<float>*>(x), ops[i], nt);
  }
  return QC_OK;
}

int qc_omp_max_threads(void) { return omp_get_max_threads(); }

const char* qc_omp_last_error(void) { return g_err.c_str(); }

}  // extern "C"
