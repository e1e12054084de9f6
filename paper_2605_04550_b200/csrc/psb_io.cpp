// Field / mask CSV export: the reference's writers (pseudospec/io.py:92-115)
// format one f-string per grid point in a Python loop, which takes minutes at C4/C5 sizes.
// These writers produce the same bytes from C++ threads.
//
// Byte compatibility with Python's f"{v:.17g}": both are correctly rounded to 17 significant
// digits with the same 'g' rules (exponent form when exp < -4 or exp >= 17, trailing zeros
// stripped, at least two exponent digits), so glibc's "%.17g" agrees for every finite value.
// The special values are spelled out here, because glibc prints a negative NaN as "-nan"
// while Python always prints "nan".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/psb200.h"

namespace {

int fmt17g(char* buf, double v) {
  if (std::isnan(v)) { std::memcpy(buf, "nan", 3); return 3; }
  if (std::isinf(v)) {
    if (v < 0) { std::memcpy(buf, "-inf", 4); return 4; }
    std::memcpy(buf, "inf", 3);
    return 3;
  }
  return std::snprintf(buf, 40, "%.17g", v);
}

std::vector<std::string> fmt_all(const double* v, int64_t n) {
  std::vector<std::string> out((size_t)n);
  char b[48];
  for (int64_t i = 0; i < n; i++) out[(size_t)i].assign(b, (size_t)fmt17g(b, v[i]));
  return out;
}

// Rows "x,y,<cell>\n" in row-major grid order (i over ys, j over xs), `cell(i, j, buf)` writes
// the third column. Grid rows are formatted in parallel blocks and written in order.
template <class Cell>
int write_rows(const char* path, const char* header, const double* xs, int64_t nx, const double* ys, int64_t ny,
               int nthreads, Cell cell) {
  if (!path || !xs || !ys || nx < 0 || ny < 0) return PSB_ERR_PARAM;
  FILE* f = std::fopen(path, "wb");
  if (!f) return PSB_ERR_IO;
  const std::vector<std::string> sx = fmt_all(xs, nx), sy = fmt_all(ys, ny);
  unsigned hw = std::thread::hardware_concurrency();
  int T = nthreads > 0 ? nthreads : (int)(hw ? hw : 1);
  if (T > 64) T = 64;
  bool ok = std::fputs(header, f) >= 0;
  const int64_t rows_per_task = 16;
  std::vector<std::string> buf((size_t)T);
  for (int64_t i0 = 0; ok && i0 < ny; i0 += rows_per_task * T) {
    std::vector<std::thread> th;
    for (int t = 0; t < T; t++) {
      const int64_t a = i0 + t * rows_per_task, b = std::min<int64_t>(ny, a + rows_per_task);
      buf[(size_t)t].clear();
      if (a >= b) continue;
      th.emplace_back([&, t, a, b]() {
        std::string& s = buf[(size_t)t];
        s.reserve((size_t)((b - a) * nx * 64));
        char c[48];
        for (int64_t i = a; i < b; i++)
          for (int64_t j = 0; j < nx; j++) {
            s += sx[(size_t)j];
            s += ',';
            s += sy[(size_t)i];
            s += ',';
            s.append(c, (size_t)cell(i * nx + j, c));
            s += '\n';
          }
      });
    }
    for (auto& x : th) x.join();
    for (int t = 0; ok && t < T; t++)
      if (!buf[(size_t)t].empty()) ok = std::fwrite(buf[(size_t)t].data(), 1, buf[(size_t)t].size(), f) == buf[(size_t)t].size();
  }
  ok = (std::fclose(f) == 0) && ok;
  return ok ? PSB_OK : PSB_ERR_IO;
}

}  // namespace

extern "C" {

int psb_write_field_csv(const char* path, const double* xs, int64_t nx, const double* ys, int64_t ny,
                        const double* log10_sigma, int32_t nthreads) {
  if (!log10_sigma && nx * ny > 0) return PSB_ERR_PARAM;
  return write_rows(path, "x,y,log10_smin\n", xs, nx, ys, ny, nthreads,
                    [&](int64_t p, char* c) { return fmt17g(c, log10_sigma[p]); });
}

int psb_write_mask_csv(const char* path, const double* xs, int64_t nx, const double* ys, int64_t ny,
                       const uint8_t* mask, int32_t nthreads) {
  if (!mask && nx * ny > 0) return PSB_ERR_PARAM;
  return write_rows(path, "x,y,flag\n", xs, nx, ys, ny, nthreads, [&](int64_t p, char* c) {
    c[0] = mask[p] ? '1' : '0';
    return 1;
  });
}

}  // extern "C"
