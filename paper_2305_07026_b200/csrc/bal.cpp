// bal.cpp — BAL dataset ingestion and convention conversion (host only, no CUDA calls).
//
// The BAL text format (Agarwal et al. 2010, the paper's datasets, Table 1): a header "M N K", K
// observations "i j u v" (centred pixels, camera i sees point j), M cameras of 9 numbers (angle-axis of R_w2c,
// t_w2c, f, k1, k2) and N points of 3 numbers, all whitespace separated.  BAL's camera looks down -z and maps
// a world point X to pixels by P = R_w2c X + t_w2c, p = -P_xy / P_z, u = f (1 + k1 |p|^2 + k2 |p|^4) p.
// The paper's model (eq. reprojection1 / ray) undistorts the observed pixel instead:
// (u, f (1 + k1' |u|^2 + k2' |u|^4)) is parallel to R^T (l - t).  daba_bal_to_paper maps one onto the other
// (reading Q15).
#include <algorithm>
#include <charconv>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <thread>
#include <vector>

#include "daba.h"

namespace daba {
void bal_to_native(const double* b, double* c);
void native_to_bal(const double* c, double* b);
}  // namespace daba

namespace {

thread_local std::string g_err;

int fail(const std::string& m) {
  g_err = m;
  return DABA_E_INVALID_ARG;
}


// line number (1-based) of byte offset `pos`
int64_t line_of(const char* b, size_t pos) {
  int64_t n = 1;
  for (size_t i = 0; i < pos; ++i) n += b[i] == '\n';
  return n;
}

template <class F>
void run_threads(int nt, F&& f) {
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(f, t);
  f(0);
  for (auto& x : th) x.join();
}

// the file's bytes, memory-mapped read-only (no copy); `n` bytes, not NUL-terminated
struct Mapped {
  const char* p = nullptr;
  size_t n = 0;
  ~Mapped() {
    if (p && n) munmap(const_cast<char*>(p), n);
  }
};

bool map_file(const char* path, Mapped& m) {
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return false;
  struct stat st;
  if (fstat(fd, &st) != 0) {
    close(fd);
    return false;
  }
  m.n = (size_t)st.st_size;
  if (m.n) {
    void* q = mmap(nullptr, m.n, PROT_READ, MAP_PRIVATE, fd, 0);
    if (q == MAP_FAILED) {
      close(fd);
      m.n = 0;
      return false;
    }
    m.p = static_cast<const char*>(q);
    madvise(q, m.n, MADV_SEQUENTIAL);
  }
  close(fd);
  return true;
}

// 1 for the whitespace bytes of the format
struct SpaceTable {
  uint8_t t[256] = {};
  SpaceTable() {
    for (unsigned char c : {' ', '\n', '\t', '\r', '\v', '\f'}) t[c] = 1;
  }
};
const SpaceTable kSpace;
inline bool is_space(char c) { return kSpace.t[(unsigned char)c]; }

// header "M N K" at the start of b; returns the offset after it or 0 on error
size_t parse_header(const char* b, size_t n, int64_t h[3]) {
  size_t p = 0;
  for (int k = 0; k < 3; ++k) {
    while (p < n && is_space(b[p])) ++p;
    auto r = std::from_chars(b + p, b + n, h[k]);
    if (r.ec != std::errc() || r.ptr == b + p || (r.ptr < b + n && !is_space(*r.ptr))) return 0;
    p = (size_t)(r.ptr - b);
  }
  return p;
}

}  // namespace

extern "C" const char* daba_bal_last_error(void) { return g_err.c_str(); }

extern "C" int daba_bal_read(const char* path, int64_t counts[3], double* cameras, double* points, int32_t* obs_cam,
                             int32_t* obs_pt, double* obs_uv) {
  g_err.clear();
  if (!path || !counts) return fail("null path or counts");
  const bool header_only = !cameras && !points && !obs_cam && !obs_pt && !obs_uv;
  if (!header_only && !(cameras && points && obs_cam && obs_pt && obs_uv)) return fail("arrays: all or none");
  const bool timing = std::getenv("DABA_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "daba_bal_read %-12s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  };
  Mapped m;
  if (!map_file(path, m)) return fail(std::string("cannot open ") + path);
  const char* b = m.p;
  const size_t n = m.n;
  int64_t h[3];
  const size_t p0 = parse_header(b, n, h);
  if (!p0) return fail("line 1: header \"num_cameras num_points num_observations\" expected");
  if (h[0] < 0 || h[1] < 0 || h[2] < 0 || h[0] > INT32_MAX || h[1] > INT32_MAX || h[2] > (INT64_C(1) << 40))
    return fail("line 1: counts out of range");
  counts[0] = h[0];
  counts[1] = h[1];
  counts[2] = h[2];
  if (header_only) return DABA_OK;
  const int64_t M = h[0], N = h[1], K = h[2];
  const int64_t T = 4 * K + 9 * M + 3 * N;  // tokens after the header
  // split the body into chunks at whitespace; pass 1 counts tokens per chunk, pass 2 parses token g into its slot
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::min(std::min<size_t>(hw, 64), 1 + (n - p0) / (1 << 20));
  std::vector<size_t> cut(nt + 1);
  cut[0] = p0;
  cut[nt] = n;
  for (int t = 1; t < nt; ++t) {
    size_t c = std::max(cut[t - 1], p0 + (n - p0) * (size_t)t / (size_t)nt);
    while (c < n && !is_space(b[c])) ++c;
    cut[t] = c;
  }
  mark("read file");
  std::vector<int64_t> ntok(nt + 1, 0);
  run_threads(nt, [&](int t) {
    int64_t c = 0;
    unsigned prev = 1;  // cut[t] is whitespace or the end of the header
    for (size_t i = cut[t]; i < cut[t + 1]; ++i) {
      const unsigned sp = kSpace.t[(unsigned char)b[i]];
      c += prev & (sp ^ 1u);
      prev = sp;
    }
    ntok[t + 1] = c;
  });
  for (int t = 0; t < nt; ++t) ntok[t + 1] += ntok[t];
  if (ntok[nt] < T) return fail("unexpected end of file: " + std::to_string(ntok[nt]) + " numbers after the header, " +
                                std::to_string(T) + " expected (4 K + 9 M + 3 N)");
  mark("count");
  // first error: (byte offset, message) per thread, the smallest offset wins
  std::vector<size_t> epos(nt, SIZE_MAX);
  std::vector<std::string> emsg(nt);
  run_threads(nt, [&](int t) {
    int64_t g = ntok[t];
    size_t i = cut[t];
    const size_t e = cut[t + 1];
    auto bad = [&](size_t at, const std::string& m) {
      epos[t] = at;
      emsg[t] = m;
    };
    while (i < e) {
      while (i < e && is_space(b[i])) ++i;
      if (i >= e) break;
      size_t j = i;
      while (j < e && !is_space(b[j])) ++j;
      if (g >= T) {
        bad(i, "trailing content after the last point");
        return;
      }
      if (g < 4 * K) {
        const int64_t q = g >> 2;
        const int f = (int)(g & 3);
        if (f < 2) {
          int64_t v;
          auto r = std::from_chars(b + i, b + j, v);
          const int64_t lim = f == 0 ? M : N;
          if (r.ec != std::errc() || r.ptr != b + j) {
            bad(i, "observation " + std::to_string(q) + ": integer index expected");
            return;
          }
          if (v < 0 || v >= lim) {
            bad(i, "observation " + std::to_string(q) + ": " + (f == 0 ? "camera" : "point") + " index " +
                       std::to_string(v) + " out of range [0, " + std::to_string(lim) + ")");
            return;
          }
          (f == 0 ? obs_cam : obs_pt)[q] = (int32_t)v;
        } else {
          auto r = std::from_chars(b + i, b + j, obs_uv[2 * q + (f - 2)]);
          if (r.ec != std::errc() || r.ptr != b + j) {
            bad(i, "observation " + std::to_string(q) + ": number expected");
            return;
          }
        }
      } else {
        const int64_t s = g - 4 * K;
        double* dst = s < 9 * M ? cameras + s : points + (s - 9 * M);
        auto r = std::from_chars(b + i, b + j, *dst);
        if (r.ec != std::errc() || r.ptr != b + j) {
          bad(i, s < 9 * M ? "camera " + std::to_string(s / 9) + ": number expected"
                           : "point " + std::to_string((s - 9 * M) / 3) + ": number expected");
          return;
        }
      }
      ++g;
      i = j;
    }
  });
  mark("parse");
  size_t best = SIZE_MAX;
  int bt = -1;
  for (int t = 0; t < nt; ++t)
    if (epos[t] < best) best = epos[t], bt = t;
  if (bt >= 0) return fail("line " + std::to_string(line_of(b, best)) + ": " + emsg[bt]);
  return DABA_OK;
}

extern "C" int daba_bal_write(const char* path, const double* cameras, int64_t M, const double* points, int64_t N,
                              const int32_t* obs_cam, const int32_t* obs_pt, const double* obs_uv, int64_t K) {
  g_err.clear();
  if (!path || M < 0 || N < 0 || K < 0 || (M && !cameras) || (N && !points) ||
      (K && (!obs_cam || !obs_pt || !obs_uv)))
    return fail("invalid arguments");
  FILE* fp = std::fopen(path, "wb");
  if (!fp) return fail(std::string("cannot open ") + path + " for writing");
  std::fprintf(fp, "%lld %lld %lld\n", (long long)M, (long long)N, (long long)K);
  for (int64_t q = 0; q < K; ++q)
    std::fprintf(fp, "%d %d %.17g %.17g\n", obs_cam[q], obs_pt[q], obs_uv[2 * q], obs_uv[2 * q + 1]);
  for (int64_t s = 0; s < 9 * M; ++s) std::fprintf(fp, "%.17g\n", cameras[s]);
  for (int64_t s = 0; s < 3 * N; ++s) std::fprintf(fp, "%.17g\n", points[s]);
  const bool ok = std::ferror(fp) == 0;
  if (std::fclose(fp) != 0 || !ok) return fail(std::string("write error on ") + path);
  return DABA_OK;
}

// BAL camera (looking down -z, forward radial distortion k1, k2 on normalised coordinates) -> the ABI camera in
// the paper's convention.  Frame: the paper's ray (u, f) must be a POSITIVE multiple of R^T (l - t); BAL's
// visible points have P_z < 0 and (u, v, f) ~ (P_x, P_y, -P_z), so observations flip v and the camera frame turns
// by S = diag(1, -1, -1) (a rotation): R^T = S R_w2c, t = the same centre -R_w2c^T t_w2c.  Intrinsics: inverting
// u = f r(|p|) p for p = u / (f g(|u|)) with g(s) = 1 + k1' s^2 + k2' s^4 gives, by series reversion,
// k1' = k1 / f^2 and k2' = (k2 - 2 k1^2) / f^4 (exact through O(s^4); reading Q15).
extern "C" int daba_bal_to_paper(double* cameras, int64_t M, double* obs_uv, int64_t K) {
  if (M < 0 || K < 0 || (M && !cameras) || (K && !obs_uv)) return DABA_E_INVALID_ARG;
  for (int64_t i = 0; i < M; ++i) {
    double* b = cameras + 9 * i;
    const double f = b[6], k1 = b[7], k2 = b[8];
    if (!(f != 0.0)) return DABA_E_INVALID_ARG;
    double c[16];
    daba::bal_to_native(b, c);  // R = R_w2c^T (rows of R_w2c as columns), t = centre
    for (int r = 0; r < 3; ++r) c[3 * r + 1] = -c[3 * r + 1], c[3 * r + 2] = -c[3 * r + 2];  // R = R_w2c^T S
    daba::native_to_bal(c, b);
    b[6] = f;
    b[7] = k1 / (f * f);
    b[8] = (k2 - 2.0 * k1 * k1) / (f * f * f * f);
  }
  for (int64_t q = 0; q < K; ++q) obs_uv[2 * q + 1] = -obs_uv[2 * q + 1];
  return DABA_OK;
}

// inverse of daba_bal_to_paper
extern "C" int daba_paper_to_bal(double* cameras, int64_t M, double* obs_uv, int64_t K) {
  if (M < 0 || K < 0 || (M && !cameras) || (K && !obs_uv)) return DABA_E_INVALID_ARG;
  for (int64_t i = 0; i < M; ++i) {
    double* b = cameras + 9 * i;
    const double f = b[6], k1p = b[7], k2p = b[8];
    if (!(f != 0.0)) return DABA_E_INVALID_ARG;
    double c[16];
    daba::bal_to_native(b, c);
    for (int r = 0; r < 3; ++r) c[3 * r + 1] = -c[3 * r + 1], c[3 * r + 2] = -c[3 * r + 2];  // S S = I
    daba::native_to_bal(c, b);
    const double k1 = k1p * f * f;
    b[6] = f;
    b[7] = k1;
    b[8] = k2p * f * f * f * f + 2.0 * k1 * k1;
  }
  for (int64_t q = 0; q < K; ++q) obs_uv[2 * q + 1] = -obs_uv[2 * q + 1];
  return DABA_OK;
}
