// OpenQASM 2.0 subset front-end (the paper's circuits arrive through QASM2
// among other front-ends, and are transpiled to the device basis {ID, SX, X, RZ, CX},
// P:684).  Grammar: OPENQASM 2.0 header; include "qelib1.inc"; qreg / creg
// (multiple registers flattened in declaration order); gate applications with constant
// parameter expressions (numbers, pi, + - * / ^, unary -, parentheses, sin/cos/sqrt/exp/ln);
// measure q -> c; reset q; barrier.  Register-wide arguments broadcast.  Not supported:
// gate / opaque definitions, if.
//
// to_basis = 1 lowers every gate to {ID, SX, X, RZ, CX} with the identities of DESIGN.md
// (global phases dropped -- they cancel in rho):
//   H = RZ(pi/2) SX RZ(pi/2); U3(t,p,l) = RZ(l) SX RZ(t+pi) SX RZ(p+pi) (time order);
//   CP(l) = RZ(l/2)_c CX RZ(-l/2)_t CX RZ(l/2)_t; CZ = H_t CX H_t; SWAP = 3 CX.
#include <cctype>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "tanq.h"
#include "tanq_internal.h"

namespace {
struct ErrSink {
  ErrSink& operator=(const std::string& m) {
    tanq::set_error(m.c_str());
    return *this;
  }
} q_err;
}

struct tanq_qasm {
  int n_qubits = 0, n_clbits = 0;
  std::vector<tanq_op> ops;
  std::vector<int32_t> measure_of_clbit;  // qubit measured into clbit c, or -1
  std::vector<std::vector<tanq_c64>> mats;  // storage of user matrices (unused by now)
};

namespace {

struct Parser {
  const std::string& s;
  size_t i = 0;
  int line = 1, col = 1;
  std::string err;
  explicit Parser(const std::string& src) : s(src) {}

  bool fail(const std::string& m) {
    if (err.empty()) err = "line " + std::to_string(line) + ":" + std::to_string(col) + ": " + m;
    return false;
  }
  void adv() {
    if (i < s.size()) {
      if (s[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
      ++i;
    }
  }
  void ws() {
    for (;;) {
      while (i < s.size() && std::isspace((unsigned char)s[i])) adv();
      if (i + 1 < s.size() && s[i] == '/' && s[i + 1] == '/') {
        while (i < s.size() && s[i] != '\n') adv();
        continue;
      }
      break;
    }
  }
  bool peek(char c) {
    ws();
    return i < s.size() && s[i] == c;
  }
  bool eat(char c) {
    if (!peek(c)) return false;
    adv();
    return true;
  }
  bool expect(char c) { return eat(c) || fail(std::string("expected '") + c + "'"); }
  std::string ident() {
    ws();
    std::string r;
    if (i < s.size() && (std::isalpha((unsigned char)s[i]) || s[i] == '_')) {
      while (i < s.size() && (std::isalnum((unsigned char)s[i]) || s[i] == '_')) {
        r += s[i];
        adv();
      }
    }
    return r;
  }
  bool number(double& v) {
    ws();
    size_t j = i;
    while (j < s.size() && (std::isdigit((unsigned char)s[j]) || s[j] == '.')) ++j;
    if (j < s.size() && (s[j] == 'e' || s[j] == 'E')) {
      ++j;
      if (j < s.size() && (s[j] == '+' || s[j] == '-')) ++j;
      while (j < s.size() && std::isdigit((unsigned char)s[j])) ++j;
    }
    if (j == i) return false;
    v = std::strtod(s.c_str() + i, nullptr);
    while (i < j) adv();
    return true;
  }
  // expr := term (('+'|'-') term)*; term := factor (('*'|'/') factor)*; factor := unary ('^' factor)?
  bool expr(double& v) {
    if (!term(v)) return false;
    for (;;) {
      if (eat('+')) {
        double w;
        if (!term(w)) return false;
        v += w;
      } else if (eat('-')) {
        double w;
        if (!term(w)) return false;
        v -= w;
      } else {
        return true;
      }
    }
  }
  bool term(double& v) {
    if (!factor(v)) return false;
    for (;;) {
      if (eat('*')) {
        double w;
        if (!factor(w)) return false;
        v *= w;
      } else if (eat('/')) {
        double w;
        if (!factor(w)) return false;
        v /= w;
      } else {
        return true;
      }
    }
  }
  bool factor(double& v) {
    if (!unary(v)) return false;
    if (eat('^')) {
      double w;
      if (!factor(w)) return false;
      v = std::pow(v, w);
    }
    return true;
  }
  bool unary(double& v) {
    if (eat('-')) {
      if (!unary(v)) return false;
      v = -v;
      return true;
    }
    if (eat('+')) return unary(v);
    if (eat('(')) return expr(v) && expect(')');
    if (number(v)) return true;
    const std::string id = ident();
    if (id == "pi") {
      v = M_PI;
      return true;
    }
    if (id == "sin" || id == "cos" || id == "tan" || id == "exp" || id == "ln" || id == "sqrt") {
      double a;
      if (!expect('(') || !expr(a) || !expect(')')) return false;
      v = id == "sin" ? std::sin(a) : id == "cos" ? std::cos(a) : id == "tan" ? std::tan(a)
        : id == "exp" ? std::exp(a) : id == "ln" ? std::log(a) : std::sqrt(a);
      return true;
    }
    return fail(id.empty() ? "expected an expression" : "unknown identifier '" + id + "'");
  }
};

struct Reg {
  int base, size;
};

void push(std::vector<tanq_op>& out, int kind, std::initializer_list<int> q, double th = 0.0) {
  tanq_op o;
  std::memset(&o, 0, sizeof(o));
  o.kind = kind;
  o.k = (int)q.size();
  int j = 0;
  for (int x : q) o.q[j++] = x;
  o.theta = th;
  o.m = nullptr;
  out.push_back(o);
}

// Emit a named gate, lowered to the basis when requested.  p[] holds up to 3 parameters.
bool emit(std::vector<tanq_op>& out, const std::string& g, const double* p, int np, const int* q,
          int nq, bool basis, std::string& err) {
  auto need = [&](int wp, int wq) {
    if (np != wp || nq != wq) {
      err = "gate '" + g + "' takes " + std::to_string(wp) + " parameter(s) and " +
            std::to_string(wq) + " qubit(s)";
      return false;
    }
    return true;
  };
  auto u3 = [&](int a, double t, double ph, double l) {
    push(out, TANQ_RZ, {a}, l);
    push(out, TANQ_SX, {a});
    push(out, TANQ_RZ, {a}, t + M_PI);
    push(out, TANQ_SX, {a});
    push(out, TANQ_RZ, {a}, ph + M_PI);
  };
  auto h = [&](int a) {
    push(out, TANQ_RZ, {a}, M_PI / 2);
    push(out, TANQ_SX, {a});
    push(out, TANQ_RZ, {a}, M_PI / 2);
  };
  static const std::map<std::string, int> one = {
      {"id", TANQ_ID}, {"x", TANQ_X}, {"y", TANQ_Y}, {"z", TANQ_Z}, {"h", TANQ_H},
      {"s", TANQ_S}, {"sdg", TANQ_SDG}, {"t", TANQ_T}, {"tdg", TANQ_TDG}, {"sx", TANQ_SX}};
  static const std::map<std::string, double> rzlike = {
      {"z", M_PI}, {"s", M_PI / 2}, {"sdg", -M_PI / 2}, {"t", M_PI / 4}, {"tdg", -M_PI / 4}};
  if (one.count(g)) {
    if (!need(0, 1)) return false;
    if (!basis || g == "id" || g == "x" || g == "sx") {
      push(out, one.at(g), {q[0]});
    } else if (g == "h") {
      h(q[0]);
    } else if (g == "y") {  // Y = i X Z: Z then X
      push(out, TANQ_RZ, {q[0]}, M_PI);
      push(out, TANQ_X, {q[0]});
    } else {
      push(out, TANQ_RZ, {q[0]}, rzlike.at(g));
    }
    return true;
  }
  if (g == "rx" || g == "ry" || g == "rz" || g == "u1" || g == "p") {
    if (!need(1, 1)) return false;
    if (!basis) {
      const int kind = g == "rx" ? TANQ_RX : g == "ry" ? TANQ_RY : TANQ_RZ;
      push(out, kind, {q[0]}, p[0]);  // u1 / p = RZ up to a global phase
    } else if (g == "rx") {
      u3(q[0], p[0], -M_PI / 2, M_PI / 2);
    } else if (g == "ry") {
      u3(q[0], p[0], 0.0, 0.0);
    } else {
      push(out, TANQ_RZ, {q[0]}, p[0]);
    }
    return true;
  }
  if (g == "u2" || g == "u3" || g == "u" || g == "U") {
    const bool two = g == "u2";
    if (!need(two ? 2 : 3, 1)) return false;
    const double t = two ? M_PI / 2 : p[0], ph = two ? p[0] : p[1], l = two ? p[1] : p[2];
    if (basis) {
      u3(q[0], t, ph, l);
    } else {  // U3 = RZ(ph) RY(t) RZ(l) up to a global phase
      push(out, TANQ_RZ, {q[0]}, l);
      push(out, TANQ_RY, {q[0]}, t);
      push(out, TANQ_RZ, {q[0]}, ph);
    }
    return true;
  }
  if (g == "cx" || g == "CX" || g == "cz" || g == "swap") {
    if (!need(0, 2)) return false;
    if (q[0] == q[1]) {
      err = "repeated qubit in '" + g + "'";
      return false;
    }
    if (g == "cx" || g == "CX") {
      push(out, TANQ_CX, {q[0], q[1]});
    } else if (!basis) {
      push(out, g == "cz" ? TANQ_CZ : TANQ_SWAP, {q[0], q[1]});
    } else if (g == "cz") {
      h(q[1]);
      push(out, TANQ_CX, {q[0], q[1]});
      h(q[1]);
    } else {
      push(out, TANQ_CX, {q[0], q[1]});
      push(out, TANQ_CX, {q[1], q[0]});
      push(out, TANQ_CX, {q[0], q[1]});
    }
    return true;
  }
  if (g == "cp" || g == "cu1" || g == "cphase") {
    if (!need(1, 2)) return false;
    if (q[0] == q[1]) {
      err = "repeated qubit in '" + g + "'";
      return false;
    }
    if (!basis) {
      push(out, TANQ_CP, {q[0], q[1]}, p[0]);
    } else {
      push(out, TANQ_RZ, {q[0]}, p[0] / 2);
      push(out, TANQ_CX, {q[0], q[1]});
      push(out, TANQ_RZ, {q[1]}, -p[0] / 2);
      push(out, TANQ_CX, {q[0], q[1]});
      push(out, TANQ_RZ, {q[1]}, p[0] / 2);
    }
    return true;
  }
  err = "unsupported gate '" + g + "'";
  return false;
}

bool parse(const std::string& src, bool basis, tanq_qasm& out, std::string& err) {
  Parser P(src);
  P.ws();
  if (P.ident() != "OPENQASM") return (err = "missing 'OPENQASM 2.0;' header", false);
  double ver;
  if (!P.number(ver) || !P.expect(';')) return (err = P.err.empty() ? "bad header" : P.err, false);
  if (std::fabs(ver - 2.0) > 1e-9) return (err = "only OPENQASM 2.0 is supported", false);
  std::map<std::string, Reg> qregs, cregs;
  for (;;) {
    P.ws();
    if (P.i >= src.size()) break;
    const int l0 = P.line, c0 = P.col;
    auto at = [&](const std::string& m) {
      err = "line " + std::to_string(l0) + ":" + std::to_string(c0) + ": " + m;
      return false;
    };
    const std::string kw = P.ident();
    if (kw.empty()) return at("expected a statement");
    if (kw == "include") {
      P.ws();
      if (!P.eat('"')) return at("expected a file name");
      std::string f;
      while (P.i < src.size() && src[P.i] != '"') {
        f += src[P.i];
        P.adv();
      }
      if (!P.eat('"') || !P.expect(';')) return at("bad include");
      if (f != "qelib1.inc") return at("only qelib1.inc can be included");
      continue;
    }
    if (kw == "qreg" || kw == "creg") {
      const std::string name = P.ident();
      double sz;
      if (name.empty() || !P.expect('[') || !P.number(sz) || !P.expect(']') || !P.expect(';'))
        return at("bad register declaration");
      auto& regs = kw == "qreg" ? qregs : cregs;
      if (qregs.count(name) || cregs.count(name)) return at("register '" + name + "' redeclared");
      int& total = kw == "qreg" ? out.n_qubits : out.n_clbits;
      regs[name] = Reg{total, (int)sz};
      total += (int)sz;
      continue;
    }
    if (kw == "gate" || kw == "opaque" || kw == "if")
      return at("'" + kw + "' is not supported (QASM2 subset)");
    // argument list helper: returns the flat indices (broadcast if a whole register)
    auto arg = [&](const std::map<std::string, Reg>& regs, std::vector<int>& idx) {
      const std::string r = P.ident();
      auto it = regs.find(r);
      if (it == regs.end()) return at("unknown register '" + r + "'");
      idx.clear();
      if (P.eat('[')) {
        double k;
        if (!P.number(k) || !P.expect(']')) return at("bad index");
        if (k < 0 || (int)k >= it->second.size) return at("index out of range for '" + r + "'");
        idx.push_back(it->second.base + (int)k);
      } else {
        for (int k = 0; k < it->second.size; ++k) idx.push_back(it->second.base + k);
      }
      return true;
    };
    if (kw == "barrier") {
      while (P.i < src.size() && src[P.i] != ';') P.adv();
      if (!P.expect(';')) return at("bad barrier");
      continue;
    }
    if (kw == "measure") {
      std::vector<int> qa, ca;
      if (!arg(qregs, qa)) return false;
      P.ws();
      if (!(P.eat('-') && P.eat('>'))) return at("expected '->'");
      if (!arg(cregs, ca)) return false;
      if (!P.expect(';')) return at("expected ';'");
      if (qa.size() != ca.size()) return at("measure register sizes differ");
      out.measure_of_clbit.resize(out.n_clbits, -1);
      for (size_t k = 0; k < qa.size(); ++k) out.measure_of_clbit[ca[k]] = qa[k];
      continue;
    }
    if (kw == "reset") {
      std::vector<int> qa;
      if (!arg(qregs, qa) || !P.expect(';')) return at("bad reset");
      for (int q : qa) push(out.ops, TANQ_RESET, {q});
      continue;
    }
    // gate application
    double p[3];
    int np = 0;
    if (P.eat('(')) {
      if (!P.peek(')')) {
        do {
          if (np == 3) return at("too many parameters");
          if (!P.expr(p[np++])) return (err = P.err, false);
        } while (P.eat(','));
      }
      if (!P.expect(')')) return (err = P.err, false);
    }
    std::vector<std::vector<int>> args;
    do {
      std::vector<int> a;
      if (!arg(qregs, a)) return false;
      args.push_back(a);
    } while (P.eat(','));
    if (!P.expect(';')) return at("expected ';'");
    size_t width = 1;
    for (auto& a : args)
      if (a.size() > 1) {
        if (width > 1 && a.size() != width) return at("register sizes differ in broadcast");
        width = a.size();
      }
    for (size_t w = 0; w < width; ++w) {
      int q[3];
      for (size_t j = 0; j < args.size() && j < 3; ++j)
        q[j] = args[j].size() == 1 ? args[j][0] : args[j][w];
      std::string e;
      if (!emit(out.ops, kw, p, np, q, (int)args.size(), basis, e)) return at(e);
    }
  }
  out.measure_of_clbit.resize(out.n_clbits, -1);
  if (out.n_qubits < 1) return (err = "no qreg declared", false);
  return true;
}

}  // namespace

extern "C" {

tanq_status tanq_qasm_parse(const char* text, int to_basis, tanq_qasm** out) {
  if (!text || !out) {
    q_err = "NULL argument";
    return TANQ_E_ARG;
  }
  *out = nullptr;
  tanq_qasm* q = new tanq_qasm();
  std::string err;
  if (!parse(std::string(text), to_basis != 0, *q, err)) {
    delete q;
    q_err = err;
    return TANQ_E_ARG;
  }
  *out = q;
  return TANQ_OK;
}

tanq_status tanq_qasm_circuit(const tanq_qasm* q, tanq_circuit* c, int* n_qubits, int* n_clbits) {
  if (!q || !c) {
    q_err = "NULL argument";
    return TANQ_E_ARG;
  }
  c->n_ops = q->ops.size();
  c->ops = q->ops.data();
  if (n_qubits) *n_qubits = q->n_qubits;
  if (n_clbits) *n_clbits = q->n_clbits;
  return TANQ_OK;
}

tanq_status tanq_qasm_measures(const tanq_qasm* q, int32_t* qubit_of_clbit) {
  if (!q || (!qubit_of_clbit && q->n_clbits)) {
    q_err = "NULL argument";
    return TANQ_E_ARG;
  }
  for (int c = 0; c < q->n_clbits; ++c) qubit_of_clbit[c] = q->measure_of_clbit[c];
  return TANQ_OK;
}

tanq_status tanq_qasm_free(tanq_qasm* q) {
  delete q;
  return TANQ_OK;
}

}  // extern "C"
