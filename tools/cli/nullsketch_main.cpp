// nullsketch_main.cpp -- command-line front end over the C ABI, compatible
// with the reference CLI's `nullspace` and `tls` subcommands
// (/root/reference/proj/tools/nullsketch_main.cpp:134-163 cmd_nullspace,
// 224-290 cmd_tls): same options, same emitted files (nullspace_W.mtx,
// tls_X.mtx, MatrixMarket dense array, %.17g), same JSON summary keys, and
// --format csv flattening.  Inputs: MatrixMarket dense arrays or headerless
// CSV (matrix.cpp:142-290 conventions).  The compute runs on the GPU through
// include/nullsketch_b200.hpp.
//
//   nullsketch_b200 [--seed S] [--out DIR] [--format json|csv] nullspace --in A.mtx
//                   [--k K (default 1) | --tol T] [--sketch KIND (default srft)] [--sketch-size S]
//                   [--certificate]
//   nullsketch_b200 [...] tls --a A.mtx --b B.mtx [--sketch KIND] [--sketch-size S]
//                   [--exact-baseline] [--allow-marginal]
#include <sys/stat.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nullsketch_b200.hpp"

namespace {

using namespace nullsketch_b200;

[[noreturn]] void io_fail(const std::string& path, long line, const std::string& what) {
  throw std::runtime_error(path + ":" + std::to_string(line) + ": " + what);
}

std::vector<std::string> tokens(const std::string& line) {
  std::vector<std::string> t;
  std::istringstream is(line);
  std::string x;
  while (is >> x) t.push_back(x);
  return t;
}

bool parse_double(const std::string& s, double& v) {
  if (s.empty()) return false;
  char* end = nullptr;
  v = std::strtod(s.c_str(), &end);
  return end && *end == '\0';
}

// "a", "a+bi", "a-bi", "bi", "i" (matrix.cpp:84-115 conventions).
bool parse_complex(std::string t, Complex& out) {
  while (!t.empty() && (t.front() == ' ' || t.front() == '\t')) t.erase(t.begin());
  while (!t.empty() && (t.back() == ' ' || t.back() == '\t')) t.pop_back();
  if (t.empty()) return false;
  if (t.back() != 'i') {
    double re;
    if (!parse_double(t, re)) return false;
    out = Complex(re, 0.0);
    return true;
  }
  t.pop_back();
  size_t split = std::string::npos;
  for (size_t i = t.size(); i-- > 1;)
    if ((t[i] == '+' || t[i] == '-') && t[i - 1] != 'e' && t[i - 1] != 'E') {
      split = i;
      break;
    }
  double re = 0.0, im;
  std::string imtok = t;
  if (split != std::string::npos) {
    if (!parse_double(t.substr(0, split), re)) return false;
    imtok = t.substr(split);
  }
  if (imtok.empty() || imtok == "+")
    im = 1.0;
  else if (imtok == "-")
    im = -1.0;
  else if (!parse_double(imtok, im))
    return false;
  out = Complex(re, im);
  return true;
}

Matrix load_matrix_market(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error(path + ": cannot open for reading");
  std::string line;
  long lineno = 1;
  if (!std::getline(in, line)) io_fail(path, 1, "empty file");
  const auto h = tokens(line);
  if (h.size() < 4 || h[0] != "%%MatrixMarket" || h[1] != "matrix") io_fail(path, 1, "expected MatrixMarket banner");
  if (h[2] != "array") io_fail(path, 1, "only dense 'array' format is supported, got '" + h[2] + "'");
  if (h[3] != "real" && h[3] != "complex") io_fail(path, 1, "unsupported field '" + h[3] + "'");
  if (h.size() >= 5 && h[4] != "general") io_fail(path, 1, "only 'general' symmetry is supported");
  const bool cplx = h[3] == "complex";
  Index rows = -1, cols = -1;
  while (rows < 0) {
    if (!std::getline(in, line)) io_fail(path, lineno + 1, "missing size line");
    ++lineno;
    if (!line.empty() && line[0] == '%') continue;
    const auto t = tokens(line);
    if (t.empty()) continue;
    double r, c;
    if (t.size() != 2 || !parse_double(t[0], r) || !parse_double(t[1], c) || r < 0 || c < 0 || r != std::floor(r) ||
        c != std::floor(c))
      io_fail(path, lineno, "expected size line 'rows cols'");
    rows = static_cast<Index>(r);
    cols = static_cast<Index>(c);
  }
  Matrix a(rows, cols, cplx ? ScalarKind::complex : ScalarKind::real);
  const Index total = rows * cols;
  Index got = 0;
  while (got < total) {
    if (!std::getline(in, line))
      io_fail(path, lineno + 1,
              "unexpected end of file, expected " + std::to_string(total) + " entries, got " + std::to_string(got));
    ++lineno;
    if (!line.empty() && line[0] == '%') continue;
    const auto t = tokens(line);
    if (t.empty()) continue;
    double x, y = 0.0;
    if (cplx ? (t.size() != 2 || !parse_double(t[0], x) || !parse_double(t[1], y))
             : (t.size() != 1 || !parse_double(t[0], x)))
      io_fail(path, lineno, cplx ? "expected 2 real tokens for a complex entry" : "expected 1 real token");
    a.set(got % rows, got / rows, Complex(x, y));  // column-major, one entry per line
    ++got;
  }
  return a;
}

Matrix load_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error(path + ": cannot open for reading");
  std::vector<std::vector<Complex>> rows;
  bool any_imag = false;
  std::string line;
  long lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.find_first_not_of(" \t") == std::string::npos) {
      if (in.peek() == std::char_traits<char>::eof()) break;
      io_fail(path, lineno, "blank line inside matrix");
    }
    std::vector<Complex> row;
    size_t start = 0;
    for (;;) {
      const size_t comma = line.find(',', start);
      const std::string tok = line.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
      Complex v;
      if (!parse_complex(tok, v)) io_fail(path, lineno, "cannot parse entry '" + tok + "'");
      any_imag = any_imag || v.imag() != 0.0;
      row.push_back(v);
      if (comma == std::string::npos) break;
      start = comma + 1;
    }
    if (!rows.empty() && row.size() != rows.front().size())
      io_fail(path, lineno,
              "row has " + std::to_string(row.size()) + " entries, expected " + std::to_string(rows.front().size()));
    rows.push_back(std::move(row));
  }
  const Index r = static_cast<Index>(rows.size()), c = r ? static_cast<Index>(rows.front().size()) : 0;
  Matrix a(r, c, any_imag ? ScalarKind::complex : ScalarKind::real);
  for (Index i = 0; i < r; ++i)
    for (Index j = 0; j < c; ++j) a.set(i, j, rows[static_cast<size_t>(i)][static_cast<size_t>(j)]);
  return a;
}

// MatrixMarket files announce themselves on the first line; anything else is CSV.
Matrix load_any(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::string first;
  std::getline(in, first);
  return first.rfind("%%MatrixMarket", 0) == 0 ? load_matrix_market(path) : load_csv(path);
}

std::string fmt(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

void save_matrix_market(const std::string& path, const Matrix& a) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error(path + ": cannot open for writing");
  out << "%%MatrixMarket matrix array " << (a.is_real() ? "real" : "complex") << " general\n";
  out << a.rows() << " " << a.cols() << "\n";
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      const Complex v = a.at(i, j);
      if (a.is_real())
        out << fmt(v.real()) << "\n";
      else
        out << fmt(v.real()) << " " << fmt(v.imag()) << "\n";
    }
  if (!out) throw std::runtime_error(path + ": write failed");
}

// ---- a small ordered JSON value (objects keep insertion order) ----------------
struct Json {
  enum Type { NUL, NUM, STR, ARR, OBJ, RAW } type = NUL;
  std::string text;                                   // NUM / STR / RAW
  std::vector<std::pair<std::string, Json>> fields;   // OBJ
  std::vector<Json> items;                            // ARR
  static Json num(double v) {
    Json j;
    if (std::isfinite(v)) {
      j.type = NUM;
      j.text = fmt(v);
    } else if (std::isinf(v)) {  // JSON has no infinity literal (nullsketch_main.cpp:58-62)
      j.type = STR;
      j.text = v > 0 ? "inf" : "-inf";
    }
    return j;
  }
  static Json integer(long long v) {
    Json j;
    j.type = RAW;
    j.text = std::to_string(v);
    return j;
  }
  static Json str(const std::string& s) {
    Json j;
    j.type = STR;
    j.text = s;
    return j;
  }
  static Json arr(const std::vector<double>& v) {
    Json j;
    j.type = ARR;
    for (double x : v) j.items.push_back(num(x));
    return j;
  }
  Json& add(const std::string& k, Json v) {
    type = OBJ;
    fields.emplace_back(k, std::move(v));
    return *this;
  }
};

std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

void dump(const Json& j, std::ostream& os, int ind, int depth) {
  const std::string pad(static_cast<size_t>(ind * (depth + 1)), ' '), end(static_cast<size_t>(ind * depth), ' ');
  switch (j.type) {
    case Json::NUL: os << "null"; break;
    case Json::NUM:
    case Json::RAW: os << j.text; break;
    case Json::STR: os << quote(j.text); break;
    case Json::ARR:
      if (j.items.empty()) {
        os << "[]";
        break;
      }
      os << "[\n";
      for (size_t i = 0; i < j.items.size(); ++i) {
        os << pad;
        dump(j.items[i], os, ind, depth + 1);
        os << (i + 1 < j.items.size() ? ",\n" : "\n");
      }
      os << end << "]";
      break;
    case Json::OBJ:
      os << "{\n";
      for (size_t i = 0; i < j.fields.size(); ++i) {
        os << pad << quote(j.fields[i].first) << ": ";
        dump(j.fields[i].second, os, ind, depth + 1);
        os << (i + 1 < j.fields.size() ? ",\n" : "\n");
      }
      os << end << "}";
      break;
  }
}

std::string compact(const Json& j) {
  std::ostringstream os;
  if (j.type == Json::ARR) {
    os << "[";
    for (size_t i = 0; i < j.items.size(); ++i) os << (i ? "," : "") << compact(j.items[i]);
    os << "]";
  } else if (j.type == Json::OBJ) {
    os << "{";
    for (size_t i = 0; i < j.fields.size(); ++i)
      os << (i ? "," : "") << quote(j.fields[i].first) << ":" << compact(j.fields[i].second);
    os << "}";
  } else {
    dump(j, os, 0, 0);
  }
  return os.str();
}

std::string csv_escape(const std::string& cell) {
  if (cell.find_first_of(",\"\n") == std::string::npos) return cell;
  std::string out = "\"";
  for (char c : cell) {
    if (c == '"') out += '"';
    out += c;
  }
  return out + "\"";
}

void flatten(const Json& j, const std::string& prefix, std::vector<std::pair<std::string, std::string>>& out) {
  if (j.type == Json::OBJ) {
    for (const auto& f : j.fields) flatten(f.second, prefix.empty() ? f.first : prefix + "." + f.first, out);
  } else if (j.type == Json::STR) {
    out.emplace_back(prefix, j.text);
  } else {
    out.emplace_back(prefix, compact(j));
  }
}

void print_summary(const Json& summary, const std::string& format) {
  if (format == "csv") {
    std::vector<std::pair<std::string, std::string>> rows;
    flatten(summary, "", rows);
    std::cout << "key,value\n";
    for (const auto& r : rows) std::cout << csv_escape(r.first) << "," << csv_escape(r.second) << "\n";
  } else {
    dump(summary, std::cout, 2, 0);
    std::cout << "\n";
  }
}

std::string prepare_out_dir(const std::string& dir) {
  std::string acc;
  for (size_t i = 0; i <= dir.size(); ++i) {  // mkdir -p
    if (i == dir.size() || dir[i] == '/') {
      if (!acc.empty()) mkdir(acc.c_str(), 0755);
    }
    if (i < dir.size()) acc += dir[i];
  }
  return dir;
}

std::string join(const std::string& dir, const std::string& file) {
  return dir.empty() || dir.back() == '/' ? dir + file : dir + "/" + file;
}

Json sketch_json(const SketchOperator& S) {
  Json j;
  j.add("kind", Json::str(to_string(S.kind())));
  j.add("size", Json::integer(S.s()));
  j.add("rows", Json::integer(S.m()));
  j.add("seed", Json::integer(static_cast<long long>(S.seed())));
  j.add("id", Json::integer(static_cast<long long>(S.id())));
  return j;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct Global {
  uint64_t seed = 1;
  std::string out_dir = ".";
  std::string format = "json";
};

int cmd_nullspace(const Global& g, const std::string& in_path, Index k, bool k_given, double tol, bool tol_given,
                  const std::string& kind_name, Index sketch_size, bool certificate) {
  if (k_given && tol_given) throw std::invalid_argument("nullspace: --k excludes --tol");
  const Matrix a = load_any(in_path);
  const Index n = a.cols();
  const SketchKind kind = sketch_kind_from_string(kind_name);
  const Index s = sketch_size > 0 ? sketch_size : default_sketch_size(kind, n);
  SketchOperator S = SketchOperator::draw(kind, s, a.rows(), g.seed);
  NullspaceResult r = tol_given ? solve_tol(a, tol, S) : solve_k(a, k, S);
  if (certificate) {
    r.residual_fro = residual_certificate(a, r.W);
    r.has_residual = true;
  }
  const std::string w_path = join(prepare_out_dir(g.out_dir), "nullspace_W.mtx");
  save_matrix_market(w_path, r.W);
  Json sm;
  sm.add("command", Json::str("nullspace"));
  sm.add("input", Json::str(in_path));
  sm.add("m", Json::integer(a.rows()));
  sm.add("n", Json::integer(n));
  sm.add("k", Json::integer(r.k));
  sm.add("tol", tol_given ? Json::num(tol) : Json());
  sm.add("sketch", sketch_json(S));
  sm.add("w_path", Json::str(w_path));
  sm.add("sketched_singular_values", Json::arr(r.sketched_singular_values));
  sm.add("residual_fro", r.has_residual ? Json::num(r.residual_fro) : Json());
  print_summary(sm, g.format);
  return 0;
}

int cmd_tls(const Global& g, const std::string& a_path, const std::string& b_path, const std::string& kind_name,
            Index sketch_size, bool exact_baseline, bool allow_marginal) {
  TlsProblem p{load_any(a_path), load_any(b_path)};
  const Index m = p.A.rows(), n = p.A.cols(), k = p.B.cols();
  const SketchKind kind = sketch_kind_from_string(kind_name);
  const Index s = sketch_size > 0 ? sketch_size : default_sketch_size(kind, n + k);
  SketchOperator S = SketchOperator::draw(kind, s, m, g.seed);
  TlsOptions opt;
  opt.allow_marginal = allow_marginal;
  auto t0 = std::chrono::steady_clock::now();
  TlsSolution sk = tls_solve_sketched(p, S, opt);
  const double sketched_seconds = seconds_since(t0);
  const std::string x_path = join(prepare_out_dir(g.out_dir), "tls_X.mtx");
  save_matrix_market(x_path, sk.X);
  Json sm;
  sm.add("command", Json::str("tls"));
  sm.add("a", Json::str(a_path));
  sm.add("b", Json::str(b_path));
  sm.add("m", Json::integer(m));
  sm.add("n", Json::integer(n));
  sm.add("k", Json::integer(k));
  sm.add("sketch", sketch_json(S));
  sm.add("x_path", Json::str(x_path));
  sm.add("tls_residual", Json::num(sk.tls_residual));
  sm.add("cond_vk2", Json::num(sk.cond_Vk2));
  sm.add("augmented_singular_values", Json::arr(sk.augmented_singular_values));
  Json timings;
  timings.add("sketched_seconds", Json::num(sketched_seconds));
  if (!exact_baseline) {
    sm.add("timings", timings);
  } else {
    auto t1 = std::chrono::steady_clock::now();
    TlsSolution ex = tls_solve_exact(p, opt);
    timings.add("exact_seconds", Json::num(seconds_since(t1)));
    sm.add("timings", timings);
    // Certified residual from an untimed re-solve (nullsketch_main.cpp:263-267).
    TlsOptions copt = opt;
    copt.certificate = true;
    const TlsSolution certified = tls_solve_sketched(p, S, copt);
    const TlsErrorMetrics met = tls_error_metrics(ex, sk);
    Json exj;
    exj.add("tls_residual", Json::num(ex.tls_residual));
    exj.add("cond_vk2", Json::num(ex.cond_Vk2));
    sm.add("exact", exj);
    sm.add("residual_certificate", Json::num(certified.residual_certificate));
    sm.add("residual_ratio", Json::num(certified.residual_certificate / ex.tls_residual));
    Json mj;
    mj.add("rel_err", Json::num(met.rel_err));
    mj.add("sin_x", Json::num(met.sin_X));
    mj.add("sin_vk", Json::num(met.sin_Vk));
    sm.add("metrics", mj);
  }
  print_summary(sm, g.format);
  return 0;
}

void usage(std::ostream& os) {
  os << "usage: nullsketch_b200 [--seed S] [--out DIR] [--format json|csv] <command> [options]\n"
        "  nullspace --in FILE [--k K | --tol T] [--sketch gaussian|srft|srdct|srht|countsketch]\n"
        "            [--sketch-size S] [--certificate]\n"
        "  tls --a FILE --b FILE [--sketch KIND] [--sketch-size S] [--exact-baseline] [--allow-marginal]\n";
}

Index to_index(const std::string& opt, const std::string& v) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (!end || *end) throw std::invalid_argument(opt + ": expected an integer, got '" + v + "'");
  return static_cast<Index>(x);
}

double to_double(const std::string& opt, const std::string& v) {
  double x;
  if (!parse_double(v, x)) throw std::invalid_argument(opt + ": expected a number, got '" + v + "'");
  return x;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  Global g;
  size_t i = 0;
  auto value = [&](const std::string& opt) -> std::string {
    if (i + 1 >= args.size()) throw std::invalid_argument(opt + " requires a value");
    return args[++i];
  };
  try {
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "-h" || a == "--help") {
        usage(std::cout);
        return 0;
      } else if (a == "--seed") {
        g.seed = static_cast<uint64_t>(std::strtoull(value(a).c_str(), nullptr, 10));
      } else if (a == "--out") {
        g.out_dir = value(a);
      } else if (a == "--format") {
        g.format = value(a);
        if (g.format != "json" && g.format != "csv") throw std::invalid_argument("--format: json or csv");
      } else {
        break;
      }
    }
    if (i >= args.size()) {
      usage(std::cerr);
      return 2;
    }
    const std::string cmd = args[i++];
    if (cmd == "nullspace") {
      std::string in, kind = "srft";  // reference defaults: k = 1, srft
      Index k = 1, size = 0;
      double tol = 0.0;
      bool k_given = false, tol_given = false, cert = false;
      for (; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a == "--in") in = value(a);
        else if (a == "--k") k = to_index(a, value(a)), k_given = true;
        else if (a == "--tol") tol = to_double(a, value(a)), tol_given = true;
        else if (a == "--sketch") kind = value(a);
        else if (a == "--sketch-size") size = to_index(a, value(a));
        else if (a == "--certificate") cert = true;
        else throw std::invalid_argument("nullspace: unknown option " + a);
      }
      if (in.empty()) throw std::invalid_argument("nullspace: --in is required");
      return cmd_nullspace(g, in, k, k_given, tol, tol_given, kind, size, cert);
    }
    if (cmd == "tls") {
      std::string pa, pb, kind = "srdct";
      Index size = 0;
      bool exact = false, marginal = false;
      for (; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a == "--a") pa = value(a);
        else if (a == "--b") pb = value(a);
        else if (a == "--sketch") kind = value(a);
        else if (a == "--sketch-size") size = to_index(a, value(a));
        else if (a == "--exact-baseline") exact = true;
        else if (a == "--allow-marginal") marginal = true;
        else throw std::invalid_argument("tls: unknown option " + a);
      }
      if (pa.empty() || pb.empty()) throw std::invalid_argument("tls: --a and --b are required");
      return cmd_tls(g, pa, pb, kind, size, exact, marginal);
    }
    throw std::invalid_argument("unknown command '" + cmd + "'");
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
