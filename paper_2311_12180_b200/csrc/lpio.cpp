// lpio.cpp — host-side LP input/output of libpdlp_b200.so (no device work).
//
//   pdlp_read_mps / pdlp_parse_mps   MPS text -> GeneralFormLp with the
//       reference reader's semantics (mps_io.hpp:163-554, docs/mps_format.md):
//       fixed / free / auto-detected columns, section order
//       NAME -> ROWS -> COLUMNS -> RHS -> [RANGES] -> [BOUNDS] -> ENDATA,
//       first N row = objective (further N rows dropped), L rows negated into
//       >= rows, ranged rows expanded into a >= pair, default bounds [0, inf)
//       applied in file order, integrality relaxed, objective-row RHS ->
//       -objective_constant, ".gz" inflated with zlib.
//   pdlp_write_solution   the `format_version 1` key-value file
//       (solution_io.hpp:70-95), doubles at max_digits10.
//
// The reader is a single pass that builds the constraint blocks row-major
// straight from per-row coefficient lists (the reference goes through
// triplets + CsrMatrix::from_triplets; the resulting CSR is identical: columns
// ascending per row, duplicates summed, exact zeros dropped).
#include <zlib.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "../../include/pdlp_b200.h"

namespace pdlp {
void set_last_error(const std::string& msg);  // capi.cu
}

struct pdlp_lp_file {
  std::string name;
  std::vector<std::string> columns;
  // G and A blocks, 64-bit indices like the reference's index_t
  std::vector<int64_t> g_off{0}, g_col, a_off{0}, a_col;
  std::vector<double> g_val, a_val, c, h, b, l, u;
  pdlp_lp view{};
};

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct ParseError : std::runtime_error {
  ParseError(int64_t line, const std::string& what)
      : std::runtime_error("mps parse error at line " + std::to_string(line) + ": " + what) {}
};

bool is_blank(char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; }

// Fixed-format field windows [begin, end) (columns 2-3, 5-12, 15-22, 25-36,
// 40-47, 50-61 in 1-based MPS terms).
constexpr int kWin[6][2] = {{1, 3}, {4, 12}, {14, 22}, {24, 36}, {39, 47}, {49, 61}};

using Tokens = std::vector<std::string_view>;

void tokens_free(std::string_view s, Tokens& out) {
  out.clear();
  size_t i = 0;
  for (;;) {
    while (i < s.size() && is_blank(s[i])) ++i;
    if (i == s.size()) return;
    const size_t b = i;
    while (i < s.size() && !is_blank(s[i])) ++i;
    if (s[b] == '$') return;  // free-format comment to end of line
    out.push_back(s.substr(b, i - b));
  }
}

void tokens_fixed(std::string_view s, Tokens& out) {
  out.clear();
  for (const auto& w : kWin) {
    if (s.size() <= size_t(w[0])) break;
    std::string_view f = s.substr(w[0], std::min(s.size(), size_t(w[1])) - w[0]);
    while (!f.empty() && is_blank(f.front())) f.remove_prefix(1);
    while (!f.empty() && is_blank(f.back())) f.remove_suffix(1);
    if (!f.empty()) out.push_back(f);
  }
}

// Every whitespace token begins inside the next unused fixed window.
bool fixed_aligned(std::string_view s) {
  int w = 0;
  size_t i = 0;
  for (;;) {
    while (i < s.size() && is_blank(s[i])) ++i;
    if (i == s.size()) return true;
    while (w < 6 && i >= size_t(kWin[w][1])) ++w;
    if (w == 6 || i < size_t(kWin[w][0])) return false;
    while (i < s.size() && !is_blank(s[i])) ++i;
    ++w;
  }
}

double number(std::string_view t, int64_t line) {
  double v = 0.0;
  const auto r = std::from_chars(t.data(), t.data() + t.size(), v);
  if (r.ec != std::errc() || r.ptr != t.data() + t.size())
    throw ParseError(line, "malformed numeric field '" + std::string(t) + "'");
  return v;
}

enum class Sec { kStart, kRows, kColumns, kRhs, kRanges, kBounds, kDone };

struct Reader {
  // rows in declaration order
  std::vector<char> kind;  // 'N', 'E', 'L', 'G'
  std::unordered_map<std::string, int64_t> row_id;
  int64_t obj = -1;
  // columns
  std::vector<std::string> cols;
  std::unordered_map<std::string, int64_t> col_id;
  // coefficients of each constraint row, file order: (column, value)
  std::vector<std::vector<std::pair<int64_t, double>>> coef;
  std::vector<double> objective;
  std::vector<double> rhs;
  std::vector<double> range;
  std::vector<char> ranged;
  double obj_rhs = 0.0;
  struct Bound {
    char op;  // 'l' lower, 'u' upper, 'x' fixed, 'f' free, 'm' -inf, 'p' +inf, 'b' binary
    int64_t col;
    double v;
  };
  std::vector<Bound> bounds;
  std::string name;

  int64_t row(std::string_view nm, int64_t line) const {
    const auto it = row_id.find(std::string(nm));
    if (it == row_id.end()) throw ParseError(line, "reference to undeclared row '" + std::string(nm) + "'");
    return it->second;
  }
  int64_t col(std::string_view nm, int64_t line) const {
    const auto it = col_id.find(std::string(nm));
    if (it == col_id.end())
      throw ParseError(line, "reference to undeclared column '" + std::string(nm) + "'");
    return it->second;
  }

  void parse(std::string_view text, int format) {
    Sec sec = Sec::kStart;
    bool integer_block = false;  // recorded by MARKER lines, relaxed downstream
    bool free_mode = format == PDLP_MPS_FREE;
    Tokens tk;
    int64_t line_no = 0;
    size_t pos = 0;
    while (pos <= text.size()) {
      const size_t nl = text.find('\n', pos);
      const size_t end = nl == std::string_view::npos ? text.size() : nl;
      std::string_view ln = text.substr(pos, end - pos);
      pos = end + 1;
      ++line_no;
      if (std::all_of(ln.begin(), ln.end(), is_blank) || ln.front() == '*') continue;
      if (ln.front() != ' ' && ln.front() != '\t') {  // section header
        tokens_free(ln, tk);
        const std::string_view head = tk.empty() ? std::string_view{} : tk[0];
        auto need = [&](bool ok, const char* what) {
          if (!ok) throw ParseError(line_no, what);
        };
        if (head == "NAME") {
          need(sec == Sec::kStart, "NAME after the header section");
          if (tk.size() > 1) name = std::string(tk[1]);
        } else if (head == "ROWS") {
          need(sec == Sec::kStart, "ROWS out of order");
          sec = Sec::kRows;
        } else if (head == "COLUMNS") {
          need(sec == Sec::kRows, "COLUMNS out of order");
          sec = Sec::kColumns;
        } else if (head == "RHS") {
          need(sec == Sec::kColumns, "RHS out of order");
          sec = Sec::kRhs;
        } else if (head == "RANGES") {
          need(sec == Sec::kRhs, "RANGES out of order");
          sec = Sec::kRanges;
        } else if (head == "BOUNDS") {
          need(sec == Sec::kRhs || sec == Sec::kRanges, "BOUNDS out of order");
          sec = Sec::kBounds;
        } else if (head == "ENDATA") {
          need(sec != Sec::kStart, "ENDATA before any data section");
          sec = Sec::kDone;
          break;
        } else {
          throw ParseError(line_no, "unknown section '" + std::string(head) + "'");
        }
        continue;
      }
      if (sec == Sec::kStart) throw ParseError(line_no, "data line before ROWS");
      if (format == PDLP_MPS_AUTO && !free_mode && !fixed_aligned(ln)) free_mode = true;
      if (format == PDLP_MPS_FIXED)
        tokens_fixed(ln, tk);
      else
        tokens_free(ln, tk);
      if (tk.empty()) continue;
      switch (sec) {
        case Sec::kRows: data_row(tk, line_no); break;
        case Sec::kColumns: data_column(tk, line_no, integer_block); break;
        case Sec::kRhs:
        case Sec::kRanges: data_rhs(tk, line_no, sec == Sec::kRhs); break;
        case Sec::kBounds: data_bound(tk, line_no); break;
        default: throw ParseError(line_no, "unexpected data line");
      }
    }
    if (sec != Sec::kDone) throw ParseError(line_no, "missing ENDATA");
    if (obj < 0) throw ParseError(line_no, "no objective (N) row declared");
  }

  void data_row(const Tokens& tk, int64_t line) {
    if (tk.size() != 2 || tk[0].size() != 1) throw ParseError(line, "ROWS line must be '<type> <name>'");
    const char t = char(std::toupper(static_cast<unsigned char>(tk[0][0])));
    if (t != 'N' && t != 'E' && t != 'L' && t != 'G')
      throw ParseError(line, "unknown row type '" + std::string(tk[0]) + "'");
    const int64_t id = int64_t(kind.size());
    if (!row_id.emplace(std::string(tk[1]), id).second)
      throw ParseError(line, "duplicate row '" + std::string(tk[1]) + "'");
    if (t == 'N' && obj < 0) obj = id;
    kind.push_back(t);
    coef.emplace_back();
    rhs.push_back(0.0);
    range.push_back(0.0);
    ranged.push_back(0);
  }

  void data_column(const Tokens& tk, int64_t line, bool& integer_block) {
    if (tk.size() >= 3 && tk[1] == "'MARKER'") {
      if (tk[2] == "'INTORG'")
        integer_block = true;
      else if (tk[2] == "'INTEND'")
        integer_block = false;
      else
        throw ParseError(line, "unknown marker '" + std::string(tk[2]) + "'");
      return;
    }
    if (tk.size() != 3 && tk.size() != 5)
      throw ParseError(line, "COLUMNS line must be '<col> <row> <value> [<row> <value>]'");
    std::string cname(tk[0]);
    auto [it, fresh] = col_id.emplace(cname, int64_t(cols.size()));
    if (fresh) {
      cols.push_back(std::move(cname));
      objective.push_back(0.0);
    }
    const int64_t j = it->second;
    for (size_t f = 1; f + 1 < tk.size(); f += 2) {
      const int64_t r = row(tk[f], line);
      const double v = number(tk[f + 1], line);
      if (r == obj)
        objective[size_t(j)] += v;
      else if (kind[size_t(r)] != 'N')  // coefficients of extra N rows vanish with the row
        coef[size_t(r)].emplace_back(j, v);
    }
  }

  void data_rhs(const Tokens& tk, int64_t line, bool is_rhs) {
    // '<set> <row> <value> [<row> <value>]'; the set name is optional (token parity)
    const size_t first = (tk.size() % 2 == 0) ? 0 : 1;
    if (tk.size() - first < 2 || (tk.size() - first) % 2 != 0)
      throw ParseError(line, "malformed RHS/RANGES line");
    for (size_t f = first; f + 1 < tk.size(); f += 2) {
      const int64_t r = row(tk[f], line);
      const double v = number(tk[f + 1], line);
      if (is_rhs) {
        rhs[size_t(r)] = v;
        if (r == obj) obj_rhs = v;
      } else {
        range[size_t(r)] = v;
        ranged[size_t(r)] = 1;
      }
    }
  }

  void data_bound(const Tokens& tk, int64_t line) {
    if (tk.empty() || tk[0].size() != 2) throw ParseError(line, "BOUNDS line must start with a two-letter type");
    std::string t(tk[0]);
    for (char& ch : t) ch = char(std::toupper(static_cast<unsigned char>(ch)));
    static const std::pair<const char*, std::pair<char, bool>> table[] = {
        {"LO", {'l', true}},  {"UP", {'u', true}},  {"FX", {'x', true}},
        {"FR", {'f', false}}, {"MI", {'m', false}}, {"PL", {'p', false}},
        {"BV", {'b', false}}, {"LI", {'l', true}},  {"UI", {'u', true}}};
    char op = 0;
    bool valued = false;
    for (const auto& e : table)
      if (t == e.first) op = e.second.first, valued = e.second.second;
    if (!op) throw ParseError(line, "unknown bound type '" + t + "'");
    // '<type> [<set>] <col> [<value>]'
    const size_t full = valued ? 4 : 3;
    size_t cf;
    if (tk.size() == full)
      cf = 2;
    else if (tk.size() + 1 == full)
      cf = 1;
    else
      throw ParseError(line, "malformed BOUNDS line");
    Bound bd{op, col(tk[cf], line), 0.0};
    if (valued) bd.v = number(tk[cf + 1], line);
    bounds.push_back(bd);
  }

  // to_general_form (mps_io.hpp:404-554)
  void build(pdlp_lp_file& f) const {
    const int64_t n = int64_t(cols.size());
    f.name = name;
    f.columns = cols;
    f.c = objective;
    f.c.resize(size_t(n), 0.0);
    std::vector<std::pair<int64_t, double>> row;
    // one output row: coefficients sorted by column, duplicates summed in file
    // order, exact zeros dropped (CsrMatrix::from_triplets, sparse_matrix.hpp:57-108)
    auto emit = [&](const std::vector<std::pair<int64_t, double>>& src, double sign,
                    std::vector<int64_t>& off, std::vector<int64_t>& cidx, std::vector<double>& val) {
      row.clear();
      for (const auto& [j, v] : src) row.emplace_back(j, sign * v);
      std::stable_sort(row.begin(), row.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      for (size_t k = 0; k < row.size();) {
        double s = row[k].second;
        size_t e = k + 1;
        for (; e < row.size() && row[e].first == row[k].first; ++e) s += row[e].second;
        if (s != 0.0) {
          cidx.push_back(row[k].first);
          val.push_back(s);
        }
        k = e;
      }
      off.push_back(int64_t(cidx.size()));
    };
    for (size_t r = 0; r < kind.size(); ++r) {
      const char k = kind[r];
      if (k == 'N') continue;
      const double q = rhs[r];
      double lo = -kInf, hi = kInf;
      if (k == 'E') {
        lo = hi = q;
        if (ranged[r]) (range[r] >= 0.0 ? hi : lo) = q + range[r];
      } else if (k == 'L') {
        hi = q;
        if (ranged[r]) lo = q - std::abs(range[r]);
      } else {  // 'G'
        lo = q;
        if (ranged[r]) hi = q + std::abs(range[r]);
      }
      if (k == 'E' && !ranged[r]) {
        emit(coef[r], 1.0, f.a_off, f.a_col, f.a_val);
        f.b.push_back(lo);
        continue;
      }
      if (lo > -kInf) {
        emit(coef[r], 1.0, f.g_off, f.g_col, f.g_val);
        f.h.push_back(1.0 * lo);
      }
      if (hi < kInf) {
        emit(coef[r], -1.0, f.g_off, f.g_col, f.g_val);
        f.h.push_back(-1.0 * hi);
      }
    }
    f.l.assign(size_t(n), 0.0);
    f.u.assign(size_t(n), kInf);
    for (const Bound& bd : bounds) {
      double& lo = f.l[size_t(bd.col)];
      double& up = f.u[size_t(bd.col)];
      switch (bd.op) {
        case 'l': lo = bd.v; break;
        case 'u': up = bd.v; break;
        case 'x': lo = up = bd.v; break;
        case 'f': lo = -kInf, up = kInf; break;
        case 'm': lo = -kInf; break;
        case 'p': up = kInf; break;
        case 'b': lo = 0.0, up = 1.0; break;
      }
    }
    for (int64_t j = 0; j < n; ++j) {
      if (f.l[size_t(j)] > f.u[size_t(j)])
        throw std::invalid_argument("infeasible bounds on variable '" + cols[size_t(j)] + "': lower " +
                                    std::to_string(f.l[size_t(j)]) + " > upper " +
                                    std::to_string(f.u[size_t(j)]));
    }
    // GeneralFormLp::validate (lp_model.hpp:45-72)
    for (int64_t j = 0; j < n; ++j) {
      const double lo = f.l[size_t(j)], up = f.u[size_t(j)];
      if (std::isnan(lo) || std::isnan(up))
        throw std::invalid_argument("lp: NaN bound on variable " + std::to_string(j));
      if (lo > up || lo == kInf || up == -kInf)
        throw std::invalid_argument("lp: empty bound interval on variable " + std::to_string(j));
    }
    for (double v : f.c)
      if (std::isnan(v)) throw std::invalid_argument("lp: NaN objective entry");

    pdlp_lp& v = f.view;
    v.inequality_matrix = pdlp_csr{int64_t(f.h.size()), n, int64_t(f.g_val.size()), f.g_off.data(),
                                   f.g_col.data(), nullptr, f.g_val.data()};
    v.equality_matrix = pdlp_csr{int64_t(f.b.size()), n, int64_t(f.a_val.size()), f.a_off.data(),
                                 f.a_col.data(), nullptr, f.a_val.data()};
    v.num_variables = n;
    v.objective = f.c.data();
    v.inequality_rhs = f.h.data();
    v.equality_rhs = f.b.data();
    v.lower = f.l.data();
    v.upper = f.u.data();
    v.objective_constant = -obj_rhs;
  }
};

std::string slurp(const std::string& path) {
  const bool gz = path.size() > 3 && path.compare(path.size() - 3, 3, ".gz") == 0;
  std::string out;
  if (gz) {
    gzFile g = gzopen(path.c_str(), "rb");
    if (!g) throw std::runtime_error("cannot open '" + path + "'");
    std::vector<char> buf(1 << 16);
    int got;
    while ((got = gzread(g, buf.data(), unsigned(buf.size()))) > 0) out.append(buf.data(), size_t(got));
    gzclose(g);
    if (got < 0) throw std::runtime_error("gzip read error in '" + path + "'");
    return out;
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open '" + path + "'");
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    pdlp::set_last_error("");
    return PDLP_OK;
  } catch (const std::invalid_argument& e) {
    pdlp::set_last_error(e.what());
    return PDLP_EINVAL;
  } catch (const std::exception& e) {
    pdlp::set_last_error(e.what());
    return PDLP_ERUNTIME;
  } catch (...) {
    pdlp::set_last_error("unknown error");
    return PDLP_ERUNTIME;
  }
}

int parse_into(std::string_view text, int32_t format, pdlp_lp_file** out) {
  if (!out) {
    pdlp::set_last_error("null argument");
    return PDLP_EINVAL;
  }
  *out = nullptr;
  return guarded([&] {
    if (format != PDLP_MPS_FIXED && format != PDLP_MPS_FREE && format != PDLP_MPS_AUTO)
      throw std::invalid_argument("mps: unknown format");
    Reader rd;
    rd.parse(text, format);
    auto* f = new pdlp_lp_file;
    try {
      rd.build(*f);
    } catch (...) {
      delete f;
      throw;
    }
    *out = f;
  });
}

std::string fmt17(double v) {
  std::ostringstream ss;
  ss.precision(std::numeric_limits<double>::max_digits10);
  ss << v;
  return ss.str();
}

const char* status_name(int s) {
  static const char* names[] = {"optimal",         "primal_infeasible", "dual_infeasible",
                                "iteration_limit", "time_limit",        "numerical_error"};
  return (s >= 0 && s < 6) ? names[s] : "unknown";
}

}  // namespace

extern "C" {

int pdlp_read_mps(const char* path, int32_t format, pdlp_lp_file** out) {
  if (!path) {
    pdlp::set_last_error("null path");
    return PDLP_EINVAL;
  }
  std::string text;
  const int rc = guarded([&] { text = slurp(path); });
  if (rc != PDLP_OK) return rc;
  return parse_into(text, format, out);
}

int pdlp_parse_mps(const char* text, int64_t length, int32_t format, pdlp_lp_file** out) {
  if (!text && length > 0) {
    pdlp::set_last_error("null text");
    return PDLP_EINVAL;
  }
  return parse_into(std::string_view(text ? text : "", size_t(length)), format, out);
}

const pdlp_lp* pdlp_lp_file_lp(const pdlp_lp_file* f) { return f ? &f->view : nullptr; }

const char* pdlp_lp_file_name(const pdlp_lp_file* f) { return f ? f->name.c_str() : nullptr; }

const char* pdlp_lp_file_column_name(const pdlp_lp_file* f, int64_t index) {
  if (!f || index < 0 || index >= int64_t(f->columns.size())) return nullptr;
  return f->columns[size_t(index)].c_str();
}

void pdlp_lp_file_free(pdlp_lp_file* f) { delete f; }

int pdlp_write_solution(const char* path, const pdlp_result_info* info, const double* x, int64_t n,
                        const double* y, int64_t m) {
  if (!path || !info) {
    pdlp::set_last_error("null argument");
    return PDLP_EINVAL;
  }
  return guarded([&] {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(std::string("cannot write '") + path + "'");
    out << "format_version 1\n";
    out << "status " << status_name(info->status) << "\n";
    out << "primal_objective " << fmt17(info->primal_objective) << "\n";
    out << "dual_objective " << fmt17(info->dual_objective) << "\n";
    out << "relative_gap " << fmt17(info->relative_gap) << "\n";
    out << "primal_residual " << fmt17(info->primal_residual_norm) << "\n";
    out << "dual_residual " << fmt17(info->dual_residual_norm) << "\n";
    out << "iterations " << info->iterations << "\n";
    out << "solve_seconds " << fmt17(info->solve_seconds) << "\n";
    if (x) {
      out << "primal_solution " << n << "\n";
      for (int64_t j = 0; j < n; ++j) out << fmt17(x[j]) << "\n";
    }
    if (y) {
      out << "dual_solution " << m << "\n";
      for (int64_t i = 0; i < m; ++i) out << fmt17(y[i]) << "\n";
    }
    if (!out) throw std::runtime_error(std::string("write failed for '") + path + "'");
  });
}

}  // extern "C"
