// Device-calibration front end: the paper drives its noise model from
// IBM backend calibration data -- per-qubit T1, T2, readout errors, per-gate error and length
// (Sec. 3.5; Table 1 uses ibmq_guadalupe).  This parses a calibration
// snapshot in the JSON schema of SPEC S:365-370 into the library's tanq_noise_model:
//
//   { "name": str, "num_qubits": int,
//     "qubits": [ {"t1_us", "t2_us", "prob_meas0_prep1", "prob_meas1_prep0",
//                  "frequency_ghz"?, "readout_length_ns"?} ],
//     "gates":  [ {"name": "id"|"sx"|"x"|"rz"|"cx", "qubits": [q] | [c, t], "error",
//                  "duration_ns", "overrot_rad"? } ],
//     "coupling_map": [[a, b], ...] }
//
// Gate error e -> depolarizing parameter p = e d / (d - 1), d = 2^k, clamped to [0, 1]
// (reading R6).  RZ entries are accepted and ignored (noiseless).
// "frequency_ghz" / "readout_length_ns" are accepted as inert metadata.  "overrot_rad" is this
// library's optional extension for the coherent over-rotation of reading R10.
// Errors: TANQ_E_ARG with the JSON path of the offending value.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tanq.h"
#include "tanq_internal.h"

namespace {

struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  double num = 0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* begin;
  std::string err;
  explicit JParser(const char* s) : p(s), begin(s) {}
  void ws() {
    while (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r') ++p;
  }
  bool fail(const std::string& m) {
    if (err.empty()) err = "offset " + std::to_string(p - begin) + ": " + m;
    return false;
  }
  bool value(JVal& v, int depth = 0) {
    if (depth > 64) return fail("nesting too deep");
    ws();
    if (*p == '{') return object(v, depth);
    if (*p == '[') return array(v, depth);
    if (*p == '"') {
      v.kind = JVal::STR;
      return string(v.str);
    }
    if (!std::strncmp(p, "true", 4)) { v.kind = JVal::BOOL; v.b = true; p += 4; return true; }
    if (!std::strncmp(p, "false", 5)) { v.kind = JVal::BOOL; v.b = false; p += 5; return true; }
    if (!std::strncmp(p, "null", 4)) { v.kind = JVal::NUL; p += 4; return true; }
    if (*p == '-' || (*p >= '0' && *p <= '9')) {
      char* end = nullptr;
      v.num = std::strtod(p, &end);
      if (end == p) return fail("bad number");
      v.kind = JVal::NUM;
      p = end;
      return true;
    }
    return fail(std::string("unexpected character '") + (*p ? std::string(1, *p) : "EOF") + "'");
  }
  bool string(std::string& out) {
    ++p;  // opening quote
    while (*p && *p != '"') {
      if (*p == '\\') {
        ++p;
        switch (*p) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u':  // keep BMP escapes as '?' -- names in this schema are ASCII
            for (int i = 0; i < 4; ++i)
              if (!*++p) return fail("truncated \\u escape");
            out += '?';
            break;
          default: return fail("bad escape");
        }
        ++p;
      } else {
        out += *p++;
      }
    }
    if (*p != '"') return fail("unterminated string");
    ++p;
    return true;
  }
  bool array(JVal& v, int depth) {
    v.kind = JVal::ARR;
    ++p;
    ws();
    if (*p == ']') { ++p; return true; }
    for (;;) {
      v.arr.emplace_back();
      if (!value(v.arr.back(), depth + 1)) return false;
      ws();
      if (*p == ',') { ++p; continue; }
      if (*p == ']') { ++p; return true; }
      return fail("expected ',' or ']'");
    }
  }
  bool object(JVal& v, int depth) {
    v.kind = JVal::OBJ;
    ++p;
    ws();
    if (*p == '}') { ++p; return true; }
    for (;;) {
      ws();
      if (*p != '"') return fail("expected a key");
      std::string k;
      if (!string(k)) return false;
      ws();
      if (*p != ':') return fail("expected ':'");
      ++p;
      v.obj.emplace_back(k, JVal());
      if (!value(v.obj.back().second, depth + 1)) return false;
      ws();
      if (*p == ',') { ++p; continue; }
      if (*p == '}') { ++p; return true; }
      return fail("expected ',' or '}'");
    }
  }
};

}  // namespace

struct tanq_device {
  std::string name;
  int n = 0;
  std::vector<tanq_qubit_cal> qubits;
  std::vector<tanq_gate_cal> gates;
  std::vector<int32_t> coupling;  // pairs
};

namespace {

tanq_status arg_err(const std::string& m) {
  tanq::set_error(m.c_str());
  return TANQ_E_ARG;
}

bool num_of(const JVal* v, double& out) {
  if (!v || v->kind != JVal::NUM || !std::isfinite(v->num)) return false;
  out = v->num;
  return true;
}

int kind_of_name(const std::string& s) {
  if (s == "id") return TANQ_ID;
  if (s == "sx") return TANQ_SX;
  if (s == "x") return TANQ_X;
  if (s == "rz") return TANQ_RZ;
  if (s == "cx") return TANQ_CX;
  return -1;
}

}  // namespace

extern "C" {

tanq_status tanq_device_parse(const char* json, tanq_device** out) {
  if (!json || !out) return arg_err("NULL argument");
  *out = nullptr;
  JParser ps(json);
  JVal root;
  if (!ps.value(root)) return arg_err("device JSON: " + ps.err);
  ps.ws();
  if (*ps.p) return arg_err("device JSON: trailing characters after the document");
  if (root.kind != JVal::OBJ) return arg_err("device JSON: $ must be an object");
  auto d = std::make_unique<tanq_device>();
  const JVal* v = root.get("name");
  if (!v || v->kind != JVal::STR) return arg_err("device JSON: $.name must be a string");
  d->name = v->str;
  double nq;
  if (!num_of(root.get("num_qubits"), nq) || nq < 1 || nq > 64 || nq != std::floor(nq))
    return arg_err("device JSON: $.num_qubits must be an integer in [1, 64]");
  d->n = (int)nq;
  v = root.get("qubits");
  if (!v || v->kind != JVal::ARR || (int)v->arr.size() != d->n)
    return arg_err("device JSON: $.qubits must be an array of num_qubits objects");
  for (int q = 0; q < d->n; ++q) {
    const JVal& o = v->arr[q];
    const std::string path = "$.qubits[" + std::to_string(q) + "]";
    if (o.kind != JVal::OBJ) return arg_err("device JSON: " + path + " must be an object");
    tanq_qubit_cal c{};
    if (!num_of(o.get("t1_us"), c.t1_us) || c.t1_us <= 0)
      return arg_err("device JSON: " + path + ".t1_us must be a positive number");
    if (!num_of(o.get("t2_us"), c.t2_us) || c.t2_us <= 0)
      return arg_err("device JSON: " + path + ".t2_us must be a positive number");
    if (c.t2_us > 2 * c.t1_us)
      return arg_err("device JSON: " + path + ": T2 > 2 T1 is unphysical (reading R8)");
    if (!num_of(o.get("prob_meas0_prep1"), c.p_meas0_prep1) || c.p_meas0_prep1 < 0 ||
        c.p_meas0_prep1 > 1)
      return arg_err("device JSON: " + path + ".prob_meas0_prep1 must be in [0, 1]");
    if (!num_of(o.get("prob_meas1_prep0"), c.p_meas1_prep0) || c.p_meas1_prep0 < 0 ||
        c.p_meas1_prep0 > 1)
      return arg_err("device JSON: " + path + ".prob_meas1_prep0 must be in [0, 1]");
    for (const char* opt : {"frequency_ghz", "readout_length_ns"}) {
      double x;
      if (o.get(opt) && !num_of(o.get(opt), x))
        return arg_err("device JSON: " + path + "." + opt + " must be a number");
    }
    d->qubits.push_back(c);
  }
  v = root.get("gates");
  if (!v || v->kind != JVal::ARR) return arg_err("device JSON: $.gates must be an array");
  for (size_t i = 0; i < v->arr.size(); ++i) {
    const JVal& o = v->arr[i];
    const std::string path = "$.gates[" + std::to_string(i) + "]";
    if (o.kind != JVal::OBJ) return arg_err("device JSON: " + path + " must be an object");
    const JVal* nmv = o.get("name");
    const int kind = nmv && nmv->kind == JVal::STR ? kind_of_name(nmv->str) : -1;
    if (kind < 0)
      return arg_err("device JSON: " + path + ".name must be one of id, sx, x, rz, cx");
    const JVal* qv = o.get("qubits");
    const int k = kind == TANQ_CX ? 2 : 1;
    if (!qv || qv->kind != JVal::ARR || (int)qv->arr.size() != k)
      return arg_err("device JSON: " + path + ".qubits must list " + std::to_string(k) +
                     " qubit(s)");
    tanq_gate_cal g{};
    g.kind = kind;
    g.k = k;
    g.q[1] = -1;
    for (int j = 0; j < k; ++j) {
      double x;
      if (!num_of(&qv->arr[j], x) || x < 0 || x >= d->n || x != std::floor(x))
        return arg_err("device JSON: " + path + ".qubits[" + std::to_string(j) +
                       "] is not a qubit of the device");
      g.q[j] = (int)x;
    }
    if (k == 2 && g.q[0] == g.q[1]) return arg_err("device JSON: " + path + ": repeated qubit");
    if (kind == TANQ_RZ) continue;  // virtual, noiseless
    double err, dur;
    if (!num_of(o.get("error"), err) || err < 0 || err > 1)
      return arg_err("device JSON: " + path + ".error must be in [0, 1]");
    if (!num_of(o.get("duration_ns"), dur) || dur < 0)
      return arg_err("device JSON: " + path + ".duration_ns must be a non-negative number");
    const double dd = (double)(1 << k);
    g.depol_p = std::min(1.0, err * dd / (dd - 1.0));  // reading R6
    g.duration_ns = dur;
    double eps = 0.0;
    if (o.get("overrot_rad") && !num_of(o.get("overrot_rad"), eps))
      return arg_err("device JSON: " + path + ".overrot_rad must be a number");
    g.overrot_rad = eps;
    d->gates.push_back(g);
  }
  v = root.get("coupling_map");
  if (v) {
    if (v->kind != JVal::ARR) return arg_err("device JSON: $.coupling_map must be an array");
    for (size_t i = 0; i < v->arr.size(); ++i) {
      const JVal& e = v->arr[i];
      double a, b;
      if (e.kind != JVal::ARR || e.arr.size() != 2 || !num_of(&e.arr[0], a) ||
          !num_of(&e.arr[1], b) || a < 0 || b < 0 || a >= d->n || b >= d->n)
        return arg_err("device JSON: $.coupling_map[" + std::to_string(i) +
                       "] must be a pair of qubits");
      d->coupling.push_back((int32_t)a);
      d->coupling.push_back((int32_t)b);
    }
  }
  *out = d.release();
  return TANQ_OK;
}

tanq_status tanq_device_noise(const tanq_device* d, tanq_noise_model* nm, int* n_qubits) {
  if (!d || !nm) return arg_err("NULL argument");
  nm->n = d->n;
  nm->order = 0;
  nm->qubits = d->qubits.data();
  nm->n_gates = d->gates.size();
  nm->gates = d->gates.data();
  if (n_qubits) *n_qubits = d->n;
  return TANQ_OK;
}

tanq_status tanq_device_coupling(const tanq_device* d, int32_t* pairs, uint64_t max, uint64_t* n) {
  if (!d || !n) return arg_err("NULL argument");
  *n = d->coupling.size() / 2;
  if (pairs)
    for (uint64_t i = 0; i < std::min<uint64_t>(max, *n); ++i) {
      pairs[2 * i] = d->coupling[2 * i];
      pairs[2 * i + 1] = d->coupling[2 * i + 1];
    }
  return TANQ_OK;
}

const char* tanq_device_name(const tanq_device* d) { return d ? d->name.c_str() : ""; }

tanq_status tanq_device_free(tanq_device* d) {
  delete d;
  return TANQ_OK;
}

}  // extern "C"
