// qasm.cpp -- openQASM 2.0 subset front end (NEXT row 4 of SURVEY 8(f)).
//
// The paper's only I/O statement: qclab++ "provides I/O through openQASM
// making it compatible with quantum hardware" (P:6).  The grammar is the
// subset SPEC S:442-495 fixes: header `OPENQASM 2.0;`, the literal
// `include "qelib1.inc";` line (accepted, not resolved), ONE `qreg`, and gate
// statements from qelib1 over that register, with constant angle expressions
// (+ - * /, unary minus, parentheses, numbers, pi).  creg / measure / reset /
// barrier / if / gate definitions / a second qreg are rejected by name.
// Errors carry line:column.  Gate names: h x y z, p|u1 -> P,
// rx ry rz, cx|CX -> CNOT, cz, cp|cu1 -> CP, swap, ccx.  Emission prints
// angles with 17 significant digits (round-trip exact for doubles).
// Host-only: no device work, no state.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "state.h"

namespace qc {
namespace {

struct Lexer {
  const char* p;
  int line = 1, col = 1;
  std::string err;
  explicit Lexer(const char* t) : p(t) {}
  void adv() {
    if (*p == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    ++p;
  }
  void skip() {
    for (;;) {
      while (*p && std::isspace((unsigned char)*p)) adv();
      if (p[0] == '/' && p[1] == '/') {
        while (*p && *p != '\n') adv();
        continue;
      }
      return;
    }
  }
  bool fail(const std::string& m) {
    if (err.empty()) err = std::to_string(line) + ":" + std::to_string(col) + ": " + m;
    return false;
  }
  bool expect(char c) {
    skip();
    if (*p != c) return fail(std::string("expected '") + c + "'");
    adv();
    return true;
  }
  bool ident(std::string& out) {
    skip();
    if (!(std::isalpha((unsigned char)*p) || *p == '_')) return fail("expected an identifier");
    out.clear();
    while (std::isalnum((unsigned char)*p) || *p == '_') {
      out += *p;
      adv();
    }
    return true;
  }
  bool integer(long long& v) {
    skip();
    if (!std::isdigit((unsigned char)*p)) return fail("expected an integer");
    v = 0;
    while (std::isdigit((unsigned char)*p)) {
      v = v * 10 + (*p - '0');
      if (v > (1ll << 40)) return fail("integer too large");
      adv();
    }
    return true;
  }
  // expr := term (('+'|'-') term)* ; term := unary (('*'|'/') unary)* ;
  // unary := '-' unary | '+' unary | primary ; primary := number | pi | '(' expr ')'
  bool expr(double& v) {
    if (!term(v)) return false;
    for (;;) {
      skip();
      if (*p != '+' && *p != '-') return true;
      const char op = *p;
      adv();
      double r;
      if (!term(r)) return false;
      v = op == '+' ? v + r : v - r;
    }
  }
  bool term(double& v) {
    if (!unary(v)) return false;
    for (;;) {
      skip();
      if (*p != '*' && *p != '/') return true;
      const char op = *p;
      adv();
      double r;
      if (!unary(r)) return false;
      if (op == '/' && r == 0.0) return fail("division by zero");
      v = op == '*' ? v * r : v / r;
    }
  }
  bool unary(double& v) {
    skip();
    if (*p == '-' || *p == '+') {
      const char op = *p;
      adv();
      if (!unary(v)) return false;
      if (op == '-') v = -v;
      return true;
    }
    return primary(v);
  }
  bool primary(double& v) {
    skip();
    if (*p == '(') {
      adv();
      if (!expr(v)) return false;
      return expect(')');
    }
    if (std::isalpha((unsigned char)*p)) {
      std::string id;
      if (!ident(id)) return false;
      if (id != "pi") return fail("unknown symbol '" + id + "' in an angle expression");
      v = 3.141592653589793238462643383279502884;
      return true;
    }
    if (std::isdigit((unsigned char)*p) || *p == '.') {
      char* end = nullptr;
      v = std::strtod(p, &end);
      if (end == p) return fail("bad number");
      while (p < end) adv();
      return true;
    }
    return fail("expected a number, pi or '('");
  }
};

struct GateName {
  const char* name;
  qc_op op;
  int nparams, nqubits;
};
const GateName kGates[] = {{"h", QC_H, 0, 1},    {"x", QC_X, 0, 1},      {"y", QC_Y, 0, 1},    {"z", QC_Z, 0, 1},
                           {"p", QC_P, 1, 1},    {"u1", QC_P, 1, 1},     {"rx", QC_RX, 1, 1},  {"ry", QC_RY, 1, 1},
                           {"rz", QC_RZ, 1, 1},  {"cx", QC_CNOT, 0, 2},  {"CX", QC_CNOT, 0, 2}, {"cz", QC_CZ, 0, 2},
                           {"cp", QC_CP, 1, 2},  {"cu1", QC_CP, 1, 2},   {"swap", QC_SWAP, 0, 2},
                           {"ccx", QC_CCX, 0, 3}};

}  // namespace
}  // namespace qc

using namespace qc;

extern "C" qc_status qc_qasm_parse(const char* text, int* n_qubits, qc_gate* ops, size_t cap, size_t* n_ops) {
  if (!text || !n_qubits || !n_ops) return fail(QC_ERR_INVALID_ARG, "qasm: NULL argument");
  Lexer L(text);
  std::vector<qc_gate> out;
  int n = -1;
  std::string reg;
  auto bad = [&]() { return fail(QC_ERR_INVALID_ARG, "qasm %s", L.err.c_str()); };
  std::string kw;
  if (!L.ident(kw) || kw != "OPENQASM") {
    L.err.clear();
    L.fail("expected 'OPENQASM 2.0;'");
    return bad();
  }
  double ver;
  if (!L.expr(ver)) return bad();
  if (ver != 2.0) {
    L.fail("only openQASM 2.0 is supported");
    return bad();
  }
  if (!L.expect(';')) return bad();
  for (;;) {
    L.skip();
    if (!*L.p) break;
    std::string id;
    if (!L.ident(id)) return bad();
    if (id == "include") {
      L.skip();
      if (*L.p != '"') {
        L.fail("expected a quoted file name");
        return bad();
      }
      L.adv();
      std::string f;
      while (*L.p && *L.p != '"' && *L.p != '\n') {
        f += *L.p;
        L.adv();
      }
      if (*L.p != '"') {
        L.fail("unterminated string");
        return bad();
      }
      L.adv();
      if (f != "qelib1.inc") {
        L.fail("only include \"qelib1.inc\" is supported");
        return bad();
      }
      if (!L.expect(';')) return bad();
      continue;
    }
    if (id == "qreg") {
      if (n >= 0) {
        L.fail("unsupported feature: a second qreg");
        return bad();
      }
      long long sz;
      if (!L.ident(reg) || !L.expect('[') || !L.integer(sz) || !L.expect(']') || !L.expect(';')) return bad();
      if (sz < 1 || sz > 62) {
        L.fail("register size must be 1..62");
        return bad();
      }
      n = (int)sz;
      continue;
    }
    if (id == "creg" || id == "measure" || id == "reset" || id == "barrier" || id == "if" || id == "gate" ||
        id == "opaque") {
      L.fail("unsupported feature: '" + id + "'");
      return bad();
    }
    const GateName* gn = nullptr;
    for (const auto& g : kGates)
      if (id == g.name) gn = &g;
    if (!gn) {
      L.fail("unsupported gate '" + id + "'");
      return bad();
    }
    if (n < 0) {
      L.fail("gate before qreg");
      return bad();
    }
    qc_gate g{};
    g.op = gn->op;
    g.ctrl_state = QC_CTRL_ONES;
    if (gn->nparams) {
      if (!L.expect('(') || !L.expr(g.theta) || !L.expect(')')) return bad();
      if (!std::isfinite(g.theta)) {
        L.fail("angle is not finite");
        return bad();
      }
    }
    for (int t = 0; t < gn->nqubits; ++t) {
      if (t && !L.expect(',')) return bad();
      std::string r;
      long long q;
      if (!L.ident(r)) return bad();
      if (r != reg) {
        L.fail("unknown register '" + r + "'");
        return bad();
      }
      if (!L.expect('[') || !L.integer(q) || !L.expect(']')) return bad();
      if (q >= n) {
        L.fail("qubit index " + std::to_string(q) + " out of range for " + reg + "[" + std::to_string(n) + "]");
        return bad();
      }
      g.qubits[t] = (int32_t)q;
    }
    for (int a = 0; a < gn->nqubits; ++a)
      for (int b = a + 1; b < gn->nqubits; ++b)
        if (g.qubits[a] == g.qubits[b]) {
          L.fail("repeated qubit operand");
          return bad();
        }
    if (!L.expect(';')) return bad();
    out.push_back(g);
  }
  if (n < 0) {
    L.fail("no qreg declared");
    return bad();
  }
  *n_qubits = n;
  *n_ops = out.size();
  if (ops) std::memcpy(ops, out.data(), std::min(cap, out.size()) * sizeof(qc_gate));
  return QC_OK;
}

extern "C" qc_status qc_qasm_emit(int n, const qc_gate* ops, size_t n_ops, char* buf, size_t cap, size_t* len) {
  if (!len || (n_ops && !ops)) return fail(QC_ERR_INVALID_ARG, "qasm: NULL argument");
  if (n < 1 || n > 62) return fail(QC_ERR_INVALID_ARG, "qasm: n must be 1..62");
  std::string s = "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[" + std::to_string(n) + "];\n";
  char num[64];
  for (size_t i = 0; i < n_ops; ++i) {
    const qc_gate& g = ops[i];
    const qc_status v = validate_gate(n, g, i);
    if (v != QC_OK) return v;
    const char* name = nullptr;
    int nq = 1;
    bool param = false;
    switch (g.op) {
      case QC_H: name = "h"; break;
      case QC_X: name = "x"; break;
      case QC_Y: name = "y"; break;
      case QC_Z: name = "z"; break;
      case QC_P: name = "u1"; param = true; break;
      case QC_RX: name = "rx"; param = true; break;
      case QC_RY: name = "ry"; param = true; break;
      case QC_RZ: name = "rz"; param = true; break;
      case QC_CNOT: name = "cx"; nq = 2; break;
      case QC_CZ: name = "cz"; nq = 2; break;
      case QC_CP: name = "cu1"; nq = 2; param = true; break;
      case QC_SWAP: name = "swap"; nq = 2; break;
      case QC_CCX: name = "ccx"; nq = 3; break;
      default: return fail(QC_ERR_UNSUPPORTED, "qasm: gate %zu (generic matrix) has no openQASM 2.0 name", i);
    }
    const int nctrl = g.op == QC_CCX ? 2 : (g.op == QC_CNOT || g.op == QC_CZ || g.op == QC_CP) ? 1 : 0;
    if (nctrl && (g.ctrl_state & ((1u << nctrl) - 1)) != ((1u << nctrl) - 1))
      return fail(QC_ERR_UNSUPPORTED, "qasm: gate %zu has a |0> control (not in qelib1)", i);
    s += name;
    if (param) {
      snprintf(num, sizeof num, "(%.17g)", g.theta);
      s += num;
    }
    for (int t = 0; t < nq; ++t) s += (t ? ",q[" : " q[") + std::to_string(g.qubits[t]) + "]";
    s += ";\n";
  }
  *len = s.size();
  if (buf && cap) {
    const size_t m = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), m);
    buf[m] = '\0';
  }
  return QC_OK;
}
