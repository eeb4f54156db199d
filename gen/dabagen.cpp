// gen/dabagen.cpp — seeded synthetic BA problems shaped like the paper's datasets.
// See dabagen.h for the contract.  Structure (SURVEY.md §8(d) "Generator v1"):
//   cameras  sequential street walk (Ladybug-like) or inward-looking rings per
//            cluster (photo collections: Venice, Trafalgar, Final), with a
//            fraction of "bridge" cameras whose id lies in one cluster's id block
//            but which sit in another cluster (long-range id edges);
//   points   created host-camera by host-camera (point ids follow camera ids,
//            which is the gather locality of real SfM exports), pixel uniform in
//            a 1600x1200 image, depth log-uniform;
//   tracks   2 + Geometric lengths with mean K/N, adjusted so the total is K;
//            each extra view is a visible candidate camera (depth > 0.5,
//            projection inside the image);
//   pixels   exact inversion of the paper's undistortion model (Newton on the
//            radius) + N(0, sigma^2) noise, a fraction of uniform outliers;
//   x^0      ground truth perturbed: R <- Exp(N(0, s_r^2 I)) R, t += N(0, s_t^2),
//            f *= 1 + N(0, s_f^2), l += N(0, (s_l * depth)^2).
// Random numbers: splitmix64-seeded xoshiro256** (portable, deterministic).
#include "dabagen.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace {

struct Rng {
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
      x += 0x9E3779B97F4A7C15ull;
      uint64_t z = x;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      s[i] = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }  // [0,1)
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
  int64_t below(int64_t n) { return (int64_t)(uniform() * (double)n); }
  double normal() {  // Box-Muller, one value per call (simple and portable)
    double u1 = uniform();
    if (u1 < 1e-300) u1 = 1e-300;
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  int64_t geometric(double p) {  // number of failures before first success
    const double u = 1.0 - uniform();
    return (int64_t)std::floor(std::log(u) / std::log(1.0 - p));
  }
};

struct V3 {
  double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline V3 normalize(V3 a) { return scale(a, 1.0 / std::sqrt(dot(a, a))); }

struct Cam {
  double R[9];  // camera -> world, row-major
  V3 t;         // centre
  double f, k1, k2;
};

inline V3 mulR(const double* R, V3 v) {
  return {R[0] * v.x + R[1] * v.y + R[2] * v.z, R[3] * v.x + R[4] * v.y + R[5] * v.z,
          R[6] * v.x + R[7] * v.y + R[8] * v.z};
}
inline V3 mulRT(const double* R, V3 v) {
  return {R[0] * v.x + R[3] * v.y + R[6] * v.z, R[1] * v.x + R[4] * v.y + R[7] * v.z,
          R[2] * v.x + R[5] * v.y + R[8] * v.z};
}

// Camera looking along `fwd` with world up (0,0,1): columns right, down, forward.
void look_rotation(V3 fwd, double* R) {
  V3 z = normalize(fwd);
  V3 up = {0, 0, 1};
  if (std::fabs(dot(z, up)) > 0.99) up = {1, 0, 0};
  V3 x = normalize(cross(z, up));
  V3 y = cross(z, x);
  R[0] = x.x; R[1] = y.x; R[2] = z.x;
  R[3] = x.y; R[4] = y.y; R[5] = z.y;
  R[6] = x.z; R[7] = y.z; R[8] = z.z;
}

void expmap(V3 w, double* A) {  // Rodrigues
  const double th2 = dot(w, w), th = std::sqrt(th2);
  double a, b;
  if (th < 1e-8) {
    a = 1.0 - th2 / 6.0;
    b = 0.5 - th2 / 24.0;
  } else {
    a = std::sin(th) / th;
    b = (1.0 - std::cos(th)) / th2;
  }
  A[0] = 1 - b * (w.y * w.y + w.z * w.z); A[1] = -a * w.z + b * w.x * w.y; A[2] = a * w.y + b * w.x * w.z;
  A[3] = a * w.z + b * w.x * w.y; A[4] = 1 - b * (w.x * w.x + w.z * w.z); A[5] = -a * w.x + b * w.y * w.z;
  A[6] = -a * w.y + b * w.x * w.z; A[7] = a * w.x + b * w.y * w.z; A[8] = 1 - b * (w.x * w.x + w.y * w.y);
}

void matmul(const double* A, const double* B, double* C) {
  double T[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) T[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
  std::memcpy(C, T, sizeof T);
}

// Angle-axis of a rotation matrix via a Shepperd quaternion (robust at 0 and pi).
V3 logmap(const double* R) {
  const double tr = R[0] + R[4] + R[8];
  double q[4];  // w x y z
  if (tr > R[0] && tr > R[4] && tr > R[8]) {
    const double s = std::sqrt(1.0 + tr) * 2;
    q[0] = 0.25 * s; q[1] = (R[7] - R[5]) / s; q[2] = (R[2] - R[6]) / s; q[3] = (R[3] - R[1]) / s;
  } else if (R[0] > R[4] && R[0] > R[8]) {
    const double s = std::sqrt(1.0 + R[0] - R[4] - R[8]) * 2;
    q[0] = (R[7] - R[5]) / s; q[1] = 0.25 * s; q[2] = (R[1] + R[3]) / s; q[3] = (R[2] + R[6]) / s;
  } else if (R[4] > R[8]) {
    const double s = std::sqrt(1.0 + R[4] - R[0] - R[8]) * 2;
    q[0] = (R[2] - R[6]) / s; q[1] = (R[1] + R[3]) / s; q[2] = 0.25 * s; q[3] = (R[5] + R[7]) / s;
  } else {
    const double s = std::sqrt(1.0 + R[8] - R[0] - R[4]) * 2;
    q[0] = (R[3] - R[1]) / s; q[1] = (R[2] + R[6]) / s; q[2] = (R[5] + R[7]) / s; q[3] = 0.25 * s;
  }
  if (q[0] < 0) for (double& v : q) v = -v;
  const double vn = std::sqrt(q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (vn < 1e-300) return {0, 0, 0};
  const double ang = 2.0 * std::atan2(vn, q[0]);
  return {q[1] / vn * ang, q[2] / vn * ang, q[3] / vn * ang};
}

constexpr double kHalfW = 800.0, kHalfH = 600.0;

// Pixel of camera-frame point q under the paper's undistortion model, or false
// when behind / outside / not invertible.  |u| = r solves
//   r = f |m| (1 + k1 r^2 + k2 r^4),  m = q_xy / q_z      (PAPER.md eq. reprojection1)
bool project(const Cam& c, V3 q, double* ux, double* uy) {
  if (q.z <= 0.5) return false;
  const double mx = q.x / q.z, my = q.y / q.z, mn = std::sqrt(mx * mx + my * my);
  if (mn * c.f > 2.0 * kHalfW) return false;
  if (mn < 1e-15) {
    *ux = 0;
    *uy = 0;
    return true;
  }
  double r = c.f * mn;
  bool ok = false;
  for (int it = 0; it < 20; ++it) {
    const double r2 = r * r;
    const double g = c.f * mn * (1.0 + c.k1 * r2 + c.k2 * r2 * r2) - r;
    const double dg = c.f * mn * (2.0 * c.k1 * r + 4.0 * c.k2 * r2 * r) - 1.0;
    if (dg >= -1e-3) return false;  // non-monotone model region
    const double step = g / dg;
    r -= step;
    if (std::fabs(step) < 1e-12 * (1.0 + r)) {
      ok = true;
      break;
    }
  }
  if (!ok || !(r >= 0)) return false;
  *ux = r * mx / mn;
  *uy = r * my / mn;
  return std::fabs(*ux) <= kHalfW && std::fabs(*uy) <= kHalfH;
}

// Camera-frame ray through pixel u (ground-truth model), normalised to z = 1.
V3 ray(const Cam& c, double ux, double uy) {
  const double s = ux * ux + uy * uy;
  const double z = c.f * (1.0 + c.k1 * s + c.k2 * s * s);
  return {ux / z, uy / z, 1.0};
}

struct Obs {
  int32_t cam, pt;
  double ux, uy;
};

}  // namespace

extern "C" void dabagen_default_params(dabagen_params* p) {
  std::memset(p, 0, sizeof *p);
  p->structure = DABAGEN_CLUSTERED;
  p->window = 30;
  p->cluster_size = 250;
  p->second_cluster_frac = 0.05;
  p->noise_px = 0.5;
  p->outlier_frac = 0.0;
  p->init_rot_deg = 0.2;
  p->init_t_sigma = 0.02;
  p->init_f_frac = 0.005;
  p->init_l_frac = 0.01;
  p->shuffle_points = 0;
  p->seed = 0x230507026ull;
}

extern "C" int dabagen_generate(const dabagen_params* p, double* cams_out, double* pts_out, int32_t* obs_cam,
                                int32_t* obs_pt, double* obs_uv, double* gt_cams_out, double* gt_pts_out,
                                int64_t* K_out) {
  if (!p || p->M <= 0 || p->N < 0 || p->K < 0 || !cams_out || (p->N > 0 && !pts_out) || !K_out) return -1;
  if (p->M > INT32_MAX || p->N > INT32_MAX) return -1;
  const int64_t M = p->M, N = p->N;
  Rng rng(p->seed);
  std::vector<Cam> cam(M);
  std::vector<int32_t> cluster_of(M, 0);
  std::vector<std::vector<int32_t>> members;  // clustered: physical members of each ring

  // ---- cameras ------------------------------------------------------------
  for (int64_t i = 0; i < M; ++i) {
    cam[i].f = rng.uniform(500.0, 1500.0);
    const double r = 1000.0;
    cam[i].k1 = rng.uniform(-1.0, 1.0) * 0.1 / (r * r);
    cam[i].k2 = rng.uniform(-1.0, 1.0) * 0.01 / (r * r * r * r);
  }
  if (p->structure == DABAGEN_SEQUENTIAL) {
    V3 pos = {0, 0, 0};
    double heading = 0;
    for (int64_t i = 0; i < M; ++i) {
      heading += rng.normal() * (5.0 * M_PI / 180.0);
      pos = add(pos, V3{std::cos(heading), std::sin(heading), 0.02 * rng.normal()});
      const double yaw = heading + rng.normal() * (10.0 * M_PI / 180.0);
      const double pitch = rng.normal() * (3.0 * M_PI / 180.0);
      V3 fwd = {std::cos(yaw) * std::cos(pitch), std::sin(yaw) * std::cos(pitch), std::sin(pitch)};
      look_rotation(fwd, cam[i].R);
      cam[i].t = pos;
    }
  } else {
    const int64_t csz = std::max<int64_t>(1, p->cluster_size);
    const int64_t C = (M + csz - 1) / csz;
    members.assign(C, {});
    std::vector<V3> centre(C);
    std::vector<double> radius(C);
    for (int64_t c = 0; c < C; ++c) {
      centre[c] = {1000.0 * (double)(c % 16), 1000.0 * (double)(c / 16), 0.0};
      radius[c] = rng.uniform(20.0, 60.0);
    }
    for (int64_t i = 0; i < M; ++i) {
      int64_t c = i / csz;
      if (C > 1 && rng.uniform() < p->second_cluster_frac) {  // bridge camera: id in block c, sits in ring c2
        int64_t c2 = rng.below(C - 1);
        if (c2 >= c) ++c2;
        c = c2;
      }
      cluster_of[i] = (int32_t)c;
      members[c].push_back((int32_t)i);
      const double phi = 6.283185307179586 * (double)(i % csz) / (double)csz + 0.01 * rng.normal();
      V3 pos = add(centre[c], V3{radius[c] * std::cos(phi), radius[c] * std::sin(phi), 2.0 * rng.normal()});
      V3 target = add(centre[c], V3{3.0 * rng.normal(), 3.0 * rng.normal(), 3.0 * rng.normal()});
      look_rotation(sub(target, pos), cam[i].R);
      cam[i].t = pos;
    }
  }

  // ---- track lengths: 2 + Geom with mean K/N, adjusted to sum K --------------
  std::vector<int64_t> L(N, 0);
  if (N > 0) {
    const double mean = (double)p->K / (double)N;
    const double pg = mean > 2.0 ? 1.0 / (mean - 1.0) : 1.0;
    int64_t S = 0;
    for (int64_t j = 0; j < N; ++j) {
      L[j] = 2 + (pg < 1.0 ? std::min<int64_t>(rng.geometric(pg), 200) : 0);
      S += L[j];
    }
    int64_t guard = 0;
    while (S > p->K && guard++ < 64 * (N + 1)) {
      const int64_t j = rng.below(N);
      if (L[j] > 2) { --L[j]; --S; }
    }
    while (S > p->K) {  // K < 2N: allow single-view tracks
      const int64_t j = rng.below(N);
      if (L[j] > 1) { --L[j]; --S; }
    }
    while (S < p->K) {
      const int64_t j = rng.below(N);
      ++L[j];
      ++S;
    }
  }

  // ---- points and tracks ---------------------------------------------------
  std::vector<V3> lgt(N);
  std::vector<double> depth(N);
  std::vector<Obs> obs;
  obs.reserve((size_t)p->K);
  int64_t carry = 0;
  std::vector<int32_t> chosen;
  const bool seq = p->structure == DABAGEN_SEQUENTIAL;
  for (int64_t j = 0; j < N; ++j) {
    const int64_t host = (j * M) / std::max<int64_t>(N, 1);
    const Cam& hc = cam[host];
    int64_t want = L[j] + carry;
    for (int attempt = 0;; ++attempt) {
      const double ux = rng.uniform(-kHalfW, kHalfW), uy = rng.uniform(-kHalfH, kHalfH);
      double z;
      if (seq) {
        z = std::exp(rng.uniform(std::log(2.0), std::log(50.0)));
      } else {
        z = std::exp(rng.uniform(std::log(10.0), std::log(80.0)));
      }
      const V3 l = add(hc.t, mulR(hc.R, scale(ray(hc, ux, uy), z)));
      chosen.clear();
      chosen.push_back((int32_t)host);
      size_t base = obs.size();
      obs.push_back({(int32_t)host, (int32_t)j, ux, uy});
      // candidate pool
      const int64_t tries = 8 * want + 16;
      for (int64_t tr = 0; tr < tries && (int64_t)chosen.size() < want; ++tr) {
        int64_t c;
        if (seq) {
          const int64_t lo = std::max<int64_t>(0, host - p->window), hi = std::min<int64_t>(M - 1, host + p->window);
          if (hi <= lo) break;
          c = lo + rng.below(hi - lo + 1);
        } else {
          const std::vector<int32_t>& mem = members[cluster_of[host]];
          if (mem.size() <= 1) break;
          c = mem[(size_t)rng.below((int64_t)mem.size())];
        }
        if (std::find(chosen.begin(), chosen.end(), (int32_t)c) != chosen.end()) continue;
        const V3 d = sub(l, cam[c].t);
        if (dot(d, d) < 1e-6) continue;
        double px, py;
        if (!project(cam[c], mulRT(cam[c].R, d), &px, &py)) continue;
        chosen.push_back((int32_t)c);
        obs.push_back({(int32_t)c, (int32_t)j, px, py});
      }
      if ((int64_t)chosen.size() >= std::min<int64_t>(2, want) || attempt >= 20) {
        lgt[j] = l;
        depth[j] = z;
        carry = want - (int64_t)chosen.size();
        break;
      }
      obs.resize(base);  // retry this point with a new pixel / depth
    }
  }
  // Remaining deficit (carry > 0) lowers K; a surplus cannot occur.
  const int64_t K = (int64_t)obs.size();

  // ---- noise and outliers ---------------------------------------------------
  for (Obs& o : obs) {
    if (p->outlier_frac > 0 && rng.uniform() < p->outlier_frac) {
      o.ux = rng.uniform(-kHalfW, kHalfW);
      o.uy = rng.uniform(-kHalfH, kHalfH);
    } else {
      o.ux += p->noise_px * rng.normal();
      o.uy += p->noise_px * rng.normal();
    }
  }

  // ---- optional point-id shuffle --------------------------------------------
  std::vector<int32_t> perm(N);
  for (int64_t j = 0; j < N; ++j) perm[j] = (int32_t)j;
  if (p->shuffle_points)
    for (int64_t j = N - 1; j > 0; --j) std::swap(perm[j], perm[rng.below(j + 1)]);

  // ---- sort observations by (camera, point) (counting sort on camera) -------
  std::vector<int64_t> cnt(M + 1, 0);
  for (const Obs& o : obs) ++cnt[o.cam + 1];
  for (int64_t i = 0; i < M; ++i) cnt[i + 1] += cnt[i];
  std::vector<Obs> sorted(obs.size());
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (const Obs& o : obs) {
      Obs q = o;
      q.pt = perm[o.pt];
      sorted[pos[o.cam]++] = q;
    }
  }
  for (int64_t i = 0; i < M; ++i)
    std::sort(sorted.begin() + cnt[i], sorted.begin() + cnt[i + 1],
              [](const Obs& a, const Obs& b) { return a.pt < b.pt; });
  for (int64_t k = 0; k < K; ++k) {
    obs_cam[k] = sorted[k].cam;
    obs_pt[k] = sorted[k].pt;
    obs_uv[2 * k] = sorted[k].ux;
    obs_uv[2 * k + 1] = sorted[k].uy;
  }

  // ---- outputs: ground truth and perturbed initial state (BAL layout) -------
  auto write_bal = [](const Cam& c, double* o) {
    double Rw2c[9] = {c.R[0], c.R[3], c.R[6], c.R[1], c.R[4], c.R[7], c.R[2], c.R[5], c.R[8]};
    const V3 aa = logmap(Rw2c);
    const V3 tw = scale(mulR(Rw2c, c.t), -1.0);
    o[0] = aa.x; o[1] = aa.y; o[2] = aa.z;
    o[3] = tw.x; o[4] = tw.y; o[5] = tw.z;
    o[6] = c.f; o[7] = c.k1; o[8] = c.k2;
  };
  const double sr = p->init_rot_deg * M_PI / 180.0;
  for (int64_t i = 0; i < M; ++i) {
    if (gt_cams_out) write_bal(cam[i], gt_cams_out + 9 * i);
    Cam c = cam[i];
    double A[9];
    expmap(V3{sr * rng.normal(), sr * rng.normal(), sr * rng.normal()}, A);
    matmul(A, cam[i].R, c.R);
    c.t = add(c.t, V3{p->init_t_sigma * rng.normal(), p->init_t_sigma * rng.normal(), p->init_t_sigma * rng.normal()});
    c.f *= 1.0 + p->init_f_frac * rng.normal();
    write_bal(c, cams_out + 9 * i);
  }
  for (int64_t j = 0; j < N; ++j) {
    const int64_t jj = perm[j];
    const V3 g = lgt[j];
    if (gt_pts_out) { gt_pts_out[3 * jj] = g.x; gt_pts_out[3 * jj + 1] = g.y; gt_pts_out[3 * jj + 2] = g.z; }
    const double s = p->init_l_frac * depth[j];
    pts_out[3 * jj] = g.x + s * rng.normal();
    pts_out[3 * jj + 1] = g.y + s * rng.normal();
    pts_out[3 * jj + 2] = g.z + s * rng.normal();
  }
  *K_out = K;
  return 0;
}
