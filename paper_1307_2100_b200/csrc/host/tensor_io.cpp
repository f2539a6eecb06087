// TENSOR v1 text I/O — the reference's on-disk format (include/tc/tensor_io.hpp:
// 9-16; writer src/tensor_io.cpp:11-27, reader :53-85), same bytes out and the
// same error messages in. The value section is formatted with std::to_chars
// (%.17g, identical to the reference's setprecision(17) stream output) in
// parallel blocks, and parsed with std::from_chars straight off the stream
// buffer: a multi-GB result is written/read at memory speed instead of
// through iostream formatting.
#include <algorithm>
#include <charconv>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <thread>

#include "tc/contract.hpp"

namespace tc {
namespace {

constexpr std::int64_t kValuesPerLine = 8;
constexpr std::int64_t kBlock = 1 << 16;  // values per formatting block (multiple of 8)

// values [lo, hi) of t as text; the separator after value i is '\n' at the end
// of every 8-value line and after the last value, else ' '
std::string format_block(const double* d, std::int64_t lo, std::int64_t hi, std::int64_t n) {
  std::string out;
  out.resize(static_cast<std::size_t>(hi - lo) * 25);
  char* p = out.data();
  char* const end = out.data() + out.size();
  for (std::int64_t i = lo; i < hi; ++i) {
    const auto r = std::to_chars(p, end, d[i], std::chars_format::general, 17);
    p = r.ptr;
    *p++ = ((i + 1) % kValuesPerLine == 0 || i + 1 == n) ? '\n' : ' ';
  }
  out.resize(static_cast<std::size_t>(p - out.data()));
  return out;
}

std::string next_line(std::istream& is) {
  std::string line;
  if (!std::getline(is, line)) throw std::runtime_error("truncated tensor file");
  return line;
}

// the text after `key` (and the spaces following it) on a header line
std::string after_key(const std::string& line, const char* key) {
  const std::string k(key);
  if (line.compare(0, k.size(), k) != 0)
    throw std::runtime_error("malformed tensor file: expected '" + k + "' line");
  std::size_t pos = k.size();
  while (pos < line.size() && line[pos] == ' ') ++pos;
  return line.substr(pos);
}

bool is_space(int c) {
  return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

// next whitespace-delimited number from the stream buffer (leading spaces
// skipped, the delimiter after it left in place)
bool next_value(std::streambuf* sb, double& v) {
  int c = sb->sgetc();
  while (c != std::char_traits<char>::eof() && is_space(c)) c = sb->snextc();
  char tok[64];
  int n = 0;
  while (c != std::char_traits<char>::eof() && !is_space(c)) {
    if (n == static_cast<int>(sizeof tok)) return false;
    tok[n++] = static_cast<char>(c);
    c = sb->snextc();
  }
  if (n == 0) return false;
  const char* b = tok;
  if (*b == '+' && n > 1) ++b;  // the stream extractor accepts an explicit sign
  const auto r = std::from_chars(b, tok + n, v);
  return r.ec == std::errc() && r.ptr == tok + n;
}

}  // namespace

void write_tensor(std::ostream& os, const Tensor& t) {
  std::string head = "TENSOR v1\nname " + (t.name().empty() ? std::string("t") : t.name()) +
                     "\nrank " + std::to_string(t.rank()) + "\nextents";
  for (int k = 0; k < t.rank(); ++k) head += " " + std::to_string(t.extent(k));
  head += "\nvariance ";
  for (int k = 0; k < t.rank(); ++k) head += variance_char(t.variance(k));
  head += "\nlayout colmajor\n";
  os << head;

  const std::int64_t n = t.size();
  const double* d = t.data();
  const std::int64_t blocks = (n + kBlock - 1) / kBlock;
  const int threads = static_cast<int>(std::min<std::int64_t>(
      blocks, std::max(1u, std::thread::hardware_concurrency())));
  if (threads <= 1) {
    for (std::int64_t b = 0; b < blocks; ++b)
      os << format_block(d, b * kBlock, std::min(n, (b + 1) * kBlock), n);
    return;
  }
  // rounds of `threads` blocks formatted concurrently, written in order
  std::vector<std::string> text(static_cast<std::size_t>(threads));
  for (std::int64_t b0 = 0; b0 < blocks; b0 += threads) {
    const int m = static_cast<int>(std::min<std::int64_t>(threads, blocks - b0));
    std::vector<std::thread> pool;
    for (int i = 0; i < m; ++i)
      pool.emplace_back([&, i] {
        const std::int64_t b = b0 + i;
        text[static_cast<std::size_t>(i)] = format_block(d, b * kBlock, std::min(n, (b + 1) * kBlock), n);
      });
    for (auto& th : pool) th.join();
    for (int i = 0; i < m; ++i) os << text[static_cast<std::size_t>(i)];
  }
}

void write_tensor_file(const std::string& path, const Tensor& t) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for writing: " + path);
  write_tensor(f, t);
}

Tensor read_tensor(std::istream& is) {
  if (next_line(is) != "TENSOR v1") throw std::runtime_error("not a TENSOR v1 file");
  const std::string name = after_key(next_line(is), "name");
  const int rank = std::stoi(after_key(next_line(is), "rank"));
  if (rank < 0) throw std::runtime_error("negative rank");

  std::vector<std::int64_t> extents;
  {
    std::istringstream es(after_key(next_line(is), "extents"));
    for (std::int64_t e; es >> e;) extents.push_back(e);
  }
  if (static_cast<int>(extents.size()) != rank)
    throw std::runtime_error("extent count does not match rank");

  const std::string vs = after_key(next_line(is), "variance");
  if (static_cast<int>(vs.size()) != rank)
    throw std::runtime_error("variance string length does not match rank");
  std::vector<Variance> variance;
  variance.reserve(vs.size());
  for (char c : vs) {
    if (c != '+' && c != '-') throw std::runtime_error("variance characters must be '+' or '-'");
    variance.push_back(c == '+' ? Variance::Up : Variance::Down);
  }
  if (after_key(next_line(is), "layout") != "colmajor")
    throw std::runtime_error("unsupported layout");

  Tensor t(std::move(extents), std::move(variance), name);
  std::streambuf* sb = is.rdbuf();
  double* d = t.data();
  for (std::int64_t i = 0; i < t.size(); ++i) {
    if (!next_value(sb, d[i])) {
      is.setstate(std::ios::failbit);
      throw std::runtime_error("truncated value section");
    }
  }
  return t;
}

Tensor read_tensor_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for reading: " + path);
  return read_tensor(f);
}

}  // namespace tc
