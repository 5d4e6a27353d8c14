// Triplet text I/O (load_triplets / save_triplets, P/include/dfc/matrix_io.hpp:125-179) for the
// input side of the path: "% m n" header (optional), then one "i j v" line per observation.
//
// The reference reads line by line through istringstreams and sorts in the ObservedMatrix
// constructor (matrix_io.hpp:38-56); at BASELINE c4 (~1e8 lines) that is minutes of serial host
// time in front of a GPU solve that takes seconds. Here the text is split at line boundaries
// into one range per host thread, each range is scanned with hand-rolled integer / strtod
// parsing, and the triplets go to column-major order by a parallel counting sort on the column
// (a per-column row sort finishes it). Semantics are the reference's:
//   * first token "%" = header; only before any data and only once ("unexpected header"),
//     dims >= 1 ("bad header dims"), nothing after them ("trailing tokens in header");
//   * a data line is "i j v" ("expected 'i j v'"), nothing after it ("trailing tokens");
//     indices after the one_based shift must be >= 0 ("negative index") and, with a header,
//     inside it (std::out_of_range, "line N: index outside declared MxN");
//   * blank lines are skipped; no header and no data is std::invalid_argument;
//   * without a header the dims are 1 + the largest indices;
//   * the first error in FILE order is the one reported (each range keeps its earliest error,
//     line numbers are resolved after the scan from the per-range line counts);
//   * duplicates are rejected after the sort (ObservedMatrix ctor): the first repeated (row,
//     col) in column-major order.
// Values print as %.17g (lossless), so save -> load is bit-exact (P/tests/test_matrix_io.cpp:99-122).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "triplet_io.hpp"

namespace dfcg {

namespace {

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f' || c == '\n'; }

int io_threads() {
  const char* e = std::getenv("DFCG_IO_THREADS");
  int t = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
  return std::max(1, std::min(t, 64));
}

// istream >> long long: optional sign, decimal digits; stops at the first other character.
bool parse_int(const char*& p, const char* end, long long& out) {
  while (p < end && is_space(*p)) ++p;
  const char* q = p;
  bool neg = false;
  if (q < end && (*q == '+' || *q == '-')) neg = *q++ == '-';
  if (q >= end || *q < '0' || *q > '9') return false;
  unsigned long long v = 0;
  bool overflow = false;
  while (q < end && *q >= '0' && *q <= '9') {
    const unsigned d = static_cast<unsigned>(*q - '0');
    if (v > (0x7fffffffffffffffULL - d) / 10) overflow = true;
    v = v * 10 + d;
    ++q;
  }
  p = q;
  if (overflow) return false;  // istream sets failbit on overflow
  out = neg ? -static_cast<long long>(v) : static_cast<long long>(v);
  return true;
}

// istream >> double (num_get): the longest prefix of the form [sign] digits [. digits]
// [e|E [sign] digits]; "inf", "nan" and hex floats are not numbers there; overflow fails.
bool parse_double(const char*& p, const char* end, double& out) {
  while (p < end && is_space(*p)) ++p;
  const char* q = p;
  if (q < end && (*q == '+' || *q == '-')) ++q;
  const char* d0 = q;
  while (q < end && *q >= '0' && *q <= '9') ++q;
  size_t digits = static_cast<size_t>(q - d0);
  if (q < end && *q == '.') {
    ++q;
    const char* f0 = q;
    while (q < end && *q >= '0' && *q <= '9') ++q;
    digits += static_cast<size_t>(q - f0);
  }
  if (digits == 0) return false;
  if (q < end && (*q == 'e' || *q == 'E')) {
    const char* e0 = q++;
    if (q < end && (*q == '+' || *q == '-')) ++q;
    const char* x0 = q;
    while (q < end && *q >= '0' && *q <= '9') ++q;
    if (q == x0) {  // "1e" / "1e+": num_get has consumed the 'e' and the conversion fails
      p = q;
      (void)e0;
      return false;
    }
  }
  char buf[64];
  const size_t len = static_cast<size_t>(q - p);
  double v;
  errno = 0;
  if (len < sizeof buf) {
    std::memcpy(buf, p, len);
    buf[len] = 0;
    v = std::strtod(buf, nullptr);
  } else {
    v = std::strtod(std::string(p, len).c_str(), nullptr);
  }
  p = q;
  if (!std::isfinite(v)) return false;  // overflow -> failbit
  out = v;
  return true;
}

bool only_space(const char* p, const char* end) {
  while (p < end && is_space(*p)) ++p;
  return p == end;
}

enum ErrKind { kNone = 0, kParse, kRange };

struct RangeResult {
  std::vector<long long> row, col;
  std::vector<double> val;
  size_t lines = 0;        // lines in the range
  ErrKind err = kNone;     // earliest error of the range
  size_t err_line = 0;     // 1-based within the range
  std::string err_msg;
  long long max_row = -1, max_col = -1;
};

// Scans [p, end): whole lines. m < 0: no header was declared.
void scan_range(const char* p, const char* end, long long base, long long m, long long n, RangeResult& r) {
  const size_t guess = static_cast<size_t>(end - p) / 12 + 16;
  r.row.reserve(guess);
  r.col.reserve(guess);
  r.val.reserve(guess);
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = nl ? nl : end;
    ++r.lines;
    const char* q = p;
    while (q < le && is_space(*q)) ++q;
    if (q < le && r.err == kNone) {
      auto fail = [&](ErrKind k, const std::string& msg) {
        r.err = k;
        r.err_line = r.lines;
        r.err_msg = msg;
      };
      // first token
      const char* t = q;
      while (t < le && !is_space(*t)) ++t;
      if (t - q == 1 && *q == '%') {
        fail(kParse, "unexpected header");  // headers are consumed before the parallel scan
      } else {
        long long i = 0, j = 0;
        double v = 0;
        const char* c = p;
        if (!parse_int(c, le, i) || !parse_int(c, le, j) || !parse_double(c, le, v)) {
          fail(kParse, "expected 'i j v'");
        } else if (!only_space(c, le)) {
          fail(kParse, "trailing tokens");
        } else {
          i -= base;
          j -= base;
          if (i < 0 || j < 0) {
            fail(kParse, "negative index");
          } else if (m >= 0 && (i >= m || j >= n)) {
            fail(kRange, "index outside declared " + std::to_string(m) + "x" + std::to_string(n));
          } else {
            r.max_row = std::max(r.max_row, i);
            r.max_col = std::max(r.max_col, j);
            r.row.push_back(i);
            r.col.push_back(j);
            r.val.push_back(v);
          }
        }
      }
    }
    if (!nl) break;
    p = nl + 1;
  }
}

template <class Fn>
void run_threads(int nt, Fn&& fn) {
  if (nt <= 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t) th.emplace_back([&, t] { fn(t); });
  for (auto& x : th) x.join();
}

}  // namespace

// Column-major order + validation of the ObservedMatrix constructor (matrix_io.hpp:38-56) for
// triplets already known to lie inside m x n with finite values: counting sort on the column
// (stable), rows sorted within each column, duplicates rejected.
void sort_column_major(long long m, long long n, std::vector<long long>& row, std::vector<long long>& col,
                       std::vector<double>& val) {
  const size_t N = val.size();
  if (N == 0) return;
  bool sorted = true;
  for (size_t i = 1; i < N && sorted; ++i)
    sorted = col[i - 1] < col[i] || (col[i - 1] == col[i] && row[i - 1] < row[i]);
  if (sorted) return;
  (void)m;
  const int nt = N < (size_t{1} << 16) ? 1 : io_threads();
  const size_t nn = static_cast<size_t>(n);
  // per-thread column histograms over contiguous input slices (stable scatter)
  const bool wide = nn * static_cast<size_t>(nt) > (size_t{1} << 28);  // histograms would not fit: one thread
  const int ht = wide ? 1 : nt;
  auto hslice = [&](int t) { return std::pair<size_t, size_t>{N * t / ht, N * (t + 1) / ht}; };
  std::vector<std::vector<size_t>> hist(static_cast<size_t>(ht));
  run_threads(ht, [&](int t) {
    auto& h = hist[static_cast<size_t>(t)];
    h.assign(nn, 0);
    const auto [a, b] = hslice(t);
    for (size_t e = a; e < b; ++e) ++h[static_cast<size_t>(col[e])];
  });
  std::vector<size_t> colptr(nn + 1, 0);
  for (size_t c = 0; c < nn; ++c) {
    size_t run = colptr[c];
    for (int t = 0; t < ht; ++t) {
      const size_t cnt = hist[static_cast<size_t>(t)][c];
      hist[static_cast<size_t>(t)][c] = run;  // this thread's first slot in column c
      run += cnt;
    }
    colptr[c + 1] = run;
  }
  std::vector<long long> r2(N), c2(N);
  std::vector<double> v2(N);
  run_threads(ht, [&](int t) {
    auto& h = hist[static_cast<size_t>(t)];
    const auto [a, b] = hslice(t);
    for (size_t e = a; e < b; ++e) {
      const size_t d = h[static_cast<size_t>(col[e])]++;
      r2[d] = row[e];
      c2[d] = col[e];
      v2[d] = val[e];
    }
  });
  // rows within each column; columns dealt to threads in contiguous ranges of ~equal entries
  run_threads(nt, [&](int t) {
    const size_t lo = N * t / nt, hi = N * (t + 1) / nt;
    size_t c0 = static_cast<size_t>(std::lower_bound(colptr.begin(), colptr.end(), lo) - colptr.begin());
    size_t c1 = static_cast<size_t>(std::lower_bound(colptr.begin(), colptr.end(), hi) - colptr.begin());
    if (t == nt - 1) c1 = nn;
    std::vector<std::pair<long long, double>> tmp;
    for (size_t c = c0; c < c1 && c < nn; ++c) {
      const size_t a = colptr[c], b = colptr[c + 1];
      bool ok = true;
      for (size_t e = a + 1; e < b && ok; ++e) ok = r2[e - 1] <= r2[e];
      if (ok) continue;
      tmp.resize(b - a);
      for (size_t e = a; e < b; ++e) tmp[e - a] = {r2[e], v2[e]};
      std::stable_sort(tmp.begin(), tmp.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t e = a; e < b; ++e) {
        r2[e] = tmp[e - a].first;
        v2[e] = tmp[e - a].second;
      }
    }
  });
  row.swap(r2);
  col.swap(c2);
  val.swap(v2);
}

void reject_duplicates(const std::vector<long long>& row, const std::vector<long long>& col) {
  for (size_t i = 1; i < row.size(); ++i)
    if (row[i - 1] == row[i] && col[i - 1] == col[i])
      throw std::invalid_argument("ObservedMatrix: duplicate entry (" + std::to_string(row[i]) + ", " +
                                  std::to_string(col[i]) + ")");
}

TripletFile load_triplets_text(const char* text, size_t len, bool one_based) {
  const long long base = one_based ? 1 : 0;
  const char* p = text;
  const char* const end = text + len;
  long long m = -1, n = -1;
  size_t lineno = 0;
  // leading blank lines and the header: sequential (a header is only legal here)
  while (p < end) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    const char* le = nl ? nl : end;
    const char* q = p;
    while (q < le && is_space(*q)) ++q;
    if (q < le) {
      const char* t = q;
      while (t < le && !is_space(*t)) ++t;
      if (!(t - q == 1 && *q == '%')) break;  // first data line: the parallel scan starts here
      if (m >= 0) throw ParseError(lineno + 1, "unexpected header");
      const char* c = t;
      long long hm = 0, hn = 0;
      if (!parse_int(c, le, hm) || !parse_int(c, le, hn) || hm < 1 || hn < 1)
        throw ParseError(lineno + 1, "bad header dims");
      if (!only_space(c, le)) throw ParseError(lineno + 1, "trailing tokens in header");
      m = hm;
      n = hn;
    }
    ++lineno;
    if (!nl) {
      p = end;
      break;
    }
    p = nl + 1;
  }
  // the body: ranges of whole lines
  const size_t body = static_cast<size_t>(end - p);
  const int nt = body < (size_t{1} << 20) ? 1 : io_threads();
  std::vector<const char*> cut(static_cast<size_t>(nt) + 1, end);
  cut[0] = p;
  for (int t = 1; t < nt; ++t) {
    const char* c = p + body * static_cast<size_t>(t) / static_cast<size_t>(nt);
    if (c < cut[static_cast<size_t>(t) - 1]) c = cut[static_cast<size_t>(t) - 1];
    const char* nl = c < end ? static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(end - c))) : nullptr;
    cut[static_cast<size_t>(t)] = nl ? nl + 1 : end;
  }
  std::vector<RangeResult> res(static_cast<size_t>(nt));
  run_threads(nt, [&](int t) {
    scan_range(cut[static_cast<size_t>(t)], cut[static_cast<size_t>(t) + 1], base, m, n, res[static_cast<size_t>(t)]);
  });
  size_t line0 = lineno;
  for (const RangeResult& r : res) {
    if (r.err == kParse) throw ParseError(line0 + r.err_line, r.err_msg);
    if (r.err == kRange) throw std::out_of_range("line " + std::to_string(line0 + r.err_line) + ": " + r.err_msg);
    line0 += r.lines;
  }
  size_t N = 0;
  long long max_row = -1, max_col = -1;
  for (const RangeResult& r : res) {
    N += r.val.size();
    max_row = std::max(max_row, r.max_row);
    max_col = std::max(max_col, r.max_col);
  }
  if (m < 0) {
    if (N == 0) throw std::invalid_argument("load_triplets: no header and no data");
    m = max_row + 1;
    n = max_col + 1;
  }
  TripletFile out;
  out.m = m;
  out.n = n;
  out.row.resize(N);
  out.col.resize(N);
  out.val.resize(N);
  {
    std::vector<size_t> off(static_cast<size_t>(nt) + 1, 0);
    for (int t = 0; t < nt; ++t) off[static_cast<size_t>(t) + 1] = off[static_cast<size_t>(t)] + res[static_cast<size_t>(t)].val.size();
    run_threads(nt, [&](int t) {
      RangeResult& r = res[static_cast<size_t>(t)];
      const size_t o = off[static_cast<size_t>(t)];
      if (r.val.empty()) return;
      std::memcpy(out.row.data() + o, r.row.data(), sizeof(long long) * r.row.size());
      std::memcpy(out.col.data() + o, r.col.data(), sizeof(long long) * r.col.size());
      std::memcpy(out.val.data() + o, r.val.data(), sizeof(double) * r.val.size());
      std::vector<long long>().swap(r.row);
      std::vector<long long>().swap(r.col);
      std::vector<double>().swap(r.val);
    });
  }
  sort_column_major(out.m, out.n, out.row, out.col, out.val);
  reject_duplicates(out.row, out.col);
  return out;
}

TripletFile load_triplets_file(const std::string& path, bool one_based) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) throw std::runtime_error("load_triplets: cannot open " + path + ": " + std::strerror(errno));
  struct stat st;
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    throw std::runtime_error("load_triplets: cannot stat " + path);
  }
  const size_t len = static_cast<size_t>(st.st_size);
  if (len == 0) {
    ::close(fd);
    return load_triplets_text("", 0, one_based);
  }
  void* map = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
  ::close(fd);
  if (map == MAP_FAILED) throw std::runtime_error("load_triplets: cannot map " + path);
  ::madvise(map, len, MADV_SEQUENTIAL);
  try {
    TripletFile out = load_triplets_text(static_cast<const char*>(map), len, one_based);
    ::munmap(map, len);
    return out;
  } catch (...) {
    ::munmap(map, len);
    throw;
  }
}

std::string format_triplets(long long m, long long n, size_t N, const long long* row, const long long* col,
                            const double* val) {
  std::string head = "% " + std::to_string(m) + " " + std::to_string(n) + "\n";
  const int nt = N < (size_t{1} << 16) ? 1 : io_threads();
  std::vector<std::string> part(static_cast<size_t>(nt));
  run_threads(nt, [&](int t) {
    const size_t a = N * static_cast<size_t>(t) / static_cast<size_t>(nt), b = N * (static_cast<size_t>(t) + 1) / static_cast<size_t>(nt);
    std::string& s = part[static_cast<size_t>(t)];
    s.reserve((b - a) * 40);
    char buf[96];
    for (size_t e = a; e < b; ++e) {
      const int k = std::snprintf(buf, sizeof buf, "%lld %lld %.17g\n", row[e], col[e], val[e]);
      s.append(buf, static_cast<size_t>(k));
    }
  });
  size_t total = head.size();
  for (const auto& s : part) total += s.size();
  std::string out;
  out.reserve(total);
  out += head;
  for (const auto& s : part) out += s;
  return out;
}

void save_triplets_file(const std::string& path, long long m, long long n, size_t N, const long long* row,
                        const long long* col, const double* val) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("save_triplets: cannot open " + path + ": " + std::strerror(errno));
  // formatted in slabs so a 1e8-entry instance does not hold its whole text in memory
  const size_t slab = size_t{1} << 22;
  bool ok = std::fprintf(f, "%% %lld %lld\n", m, n) > 0;
  for (size_t a = 0; a < N && ok; a += slab) {
    const size_t cnt = std::min(slab, N - a);
    const std::string s = format_triplets(m, n, cnt, row + a, col + a, val + a);
    const size_t skip = s.find('\n') + 1;  // the slab's own header line
    ok = std::fwrite(s.data() + skip, 1, s.size() - skip, f) == s.size() - skip;
  }
  if (std::fclose(f) != 0) ok = false;
  if (!ok) throw std::runtime_error("save_triplets: write to " + path + " failed");
}

}  // namespace dfcg
