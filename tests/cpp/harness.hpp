// Minimal test harness for the C++ parity suites (the reference uses doctest,
// which is not in this image): TEST_CASE registers a function, CHECK records
// failures, main() runs all cases and returns the failure count.
#pragma once
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace th {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline int& failures() {
  static int f = 0;
  return f;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, what.c_str());
}
}  // namespace th

#define TH_CAT2(a, b) a##b
#define TH_CAT(a, b) TH_CAT2(a, b)
#define TEST_CASE(name)                                             \
  static void TH_CAT(th_case_, __LINE__)();                         \
  static th::Reg TH_CAT(th_reg_, __LINE__)(name, TH_CAT(th_case_, __LINE__)); \
  static void TH_CAT(th_case_, __LINE__)()
#define CHECK(x) \
  do { if (!(x)) th::fail(__FILE__, __LINE__, #x); } while (0)
#define CHECK_FALSE(x) CHECK(!(x))
#define REQUIRE(x) \
  do { if (!(x)) { th::fail(__FILE__, __LINE__, #x); return; } } while (0)
#define CHECK_THROWS_AS(expr, type)                                          \
  do {                                                                       \
    bool th_ok = false;                                                      \
    try { (void)(expr); } catch (const type&) { th_ok = true; } catch (...) {} \
    if (!th_ok) th::fail(__FILE__, __LINE__, "throws " #type ": " #expr);   \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, msg, type)                                \
  do {                                                                       \
    bool th_ok = false;                                                      \
    try { (void)(expr); } catch (const type& e) { th_ok = std::string(e.what()) == (msg); } \
    catch (...) {}                                                           \
    if (!th_ok) th::fail(__FILE__, __LINE__, "throws '" msg "': " #expr);   \
  } while (0)

#define TH_MAIN                                                        \
  int main() {                                                         \
    for (auto& c : th::cases()) {                                      \
      const int before = th::failures();                               \
      try { c.fn(); } catch (const std::exception& e) {                \
        th::fail(__FILE__, 0, std::string(c.name) + " threw: " + e.what()); \
      }                                                                \
      std::printf("%s %s\n", th::failures() == before ? "ok  " : "FAIL", c.name); \
    }                                                                  \
    std::printf("%d failure(s) in %zu cases\n", th::failures(), th::cases().size()); \
    return th::failures() ? 1 : 0;                                     \
  }
