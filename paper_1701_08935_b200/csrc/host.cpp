// Host-side setup that stays on the CPU by design (BASELINE.json north_star:
// "ordering and symbolic analysis remain host-side setup"):
//   - reverse Cuthill-McKee ordering (rcm.hpp:33-147),
//   - the reference's bit-reproducible Gaussian block + MGS (dense.hpp:181-229).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <random>
#include <thread>
#include <vector>

#include "host.hpp"

namespace zolo {

namespace {

// BFS levels from root; farthest node with ties to smaller degree then index
// (rcm.hpp:33-62).
int64_t bfs_far_node(int64_t n, const int64_t* rp, const int64_t* ci, int64_t root, std::vector<int64_t>& level,
                     std::vector<int64_t>& queue) {
  level.assign(n, -1);
  queue.clear();
  queue.push_back(root);
  level[root] = 0;
  int64_t far = root, far_level = 0;
  for (size_t h = 0; h < queue.size(); ++h) {
    const int64_t u = queue[h];
    for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
      const int64_t v = ci[k];
      if (v != u && level[v] < 0) {
        level[v] = level[u] + 1;
        queue.push_back(v);
        if (level[v] > far_level) {
          far_level = level[v];
          far = v;
        } else if (level[v] == far_level) {
          const int64_t du = rp[far + 1] - rp[far], dv = rp[v + 1] - rp[v];
          if (dv < du || (dv == du && v < far)) far = v;
        }
      }
    }
  }
  return far;
}

}  // namespace

void rcm_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm) {
  const auto degree = [rp](int64_t v) { return rp[v + 1] - rp[v]; };
  std::vector<char> visited(n, 0);
  std::vector<int64_t> level, queue, nbrs, order;
  order.reserve(n);
  while (static_cast<int64_t>(order.size()) < n) {
    int64_t root = n, best = std::numeric_limits<int64_t>::max();
    for (int64_t v = 0; v < n; ++v)
      if (!visited[v] && degree(v) < best) {
        best = degree(v);
        root = v;
      }
    for (int it = 0; it < 2; ++it) root = bfs_far_node(n, rp, ci, root, level, queue);
    std::vector<int64_t> q;
    q.push_back(root);
    visited[root] = 1;
    for (size_t h = 0; h < q.size(); ++h) {
      const int64_t u = q[h];
      order.push_back(u);
      nbrs.clear();
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
        const int64_t v = ci[k];
        if (v != u && !visited[v]) {
          visited[v] = 1;
          nbrs.push_back(v);
        }
      }
      std::sort(nbrs.begin(), nbrs.end(), [&](int64_t x, int64_t y) {
        const int64_t dx = degree(x), dy = degree(y);
        return dx < dy || (dx == dy && x < y);
      });
      for (int64_t v : nbrs) q.push_back(v);
    }
  }
  std::reverse(order.begin(), order.end());
  std::copy(order.begin(), order.end(), perm);
}

int64_t bandwidth_under(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* perm) {
  std::vector<int64_t> pos(n);
  for (int64_t k = 0; k < n; ++k) pos[perm[k]] = k;
  int64_t bw = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) { const int64_t d = pos[i] - pos[ci[k]]; bw = std::max<int64_t>(bw, d < 0 ? -d : d); }
  return bw;
}

int64_t profile_under(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* perm) {
  std::vector<int64_t> pos(n), lowest(n);
  for (int64_t k = 0; k < n; ++k) pos[perm[k]] = k;
  for (int64_t i = 0; i < n; ++i) lowest[pos[i]] = pos[i];
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t a = std::max(pos[i], pos[ci[k]]), b = std::min(pos[i], pos[ci[k]]);
      lowest[a] = std::min(lowest[a], b);
    }
  int64_t prof = 0;
  for (int64_t i = 0; i < n; ++i) prof += i - lowest[i];
  return prof;
}

namespace {
double uniform_unit(std::mt19937_64& rng) { return (static_cast<double>(rng() >> 11) + 0.5) * 0x1.0p-53; }
double gaussian(std::mt19937_64& rng) {
  const double u1 = uniform_unit(rng);
  const double u2 = uniform_unit(rng);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

template <class S>
double abs2(S x) {
  return std::norm(std::complex<double>(x));
}
inline double conj_s(double x) { return x; }
inline std::complex<double> conj_s(std::complex<double> x) { return std::conj(x); }

template <class S>
bool mgs(S* q, int64_t n, int64_t k) {
  for (int64_t j = 0; j < k; ++j) {
    S* qj = q + j * n;
    double before = 0;
    for (int64_t t = 0; t < n; ++t) before += abs2(qj[t]);
    before = std::sqrt(before);
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t i = 0; i < j; ++i) {
        const S* qi = q + i * n;
        S h(0);
        for (int64_t t = 0; t < n; ++t) h += conj_s(qi[t]) * qj[t];
        for (int64_t t = 0; t < n; ++t) qj[t] -= h * qi[t];
      }
    double nrm = 0;
    for (int64_t t = 0; t < n; ++t) nrm += abs2(qj[t]);
    nrm = std::sqrt(nrm);
    if (!(nrm > 1e-14 * std::max(1.0, before))) return false;
    for (int64_t t = 0; t < n; ++t) qj[t] = qj[t] * S(1.0 / nrm);
  }
  return true;
}
}  // namespace

void uniform_stream(uint64_t seed, int64_t n, double* out) {
  // hamiltonian.hpp:52 convention: raw mt19937_64 bits, (x >> 11) 2^-53 in [0,1)
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
}

// The raw mt19937_64 stream is sequential by definition (dense.hpp:193-208 draws in column
// order from one generator), the Box-Muller transform of each pair of draws is not: the stream is
// produced block by block on the calling thread and transformed by a few host threads, each
// Gaussian by the same expression as the serial form (bit-identical output).
namespace {
void gaussian_fill(std::mt19937_64& rng, int64_t count, double* out) {
  // ~16 blocks per call, between 64 Ki and 1 Mi Gaussians each (a block's raw draws overlap the
  // transform of the block before)
  const int64_t BLK = std::min<int64_t>(int64_t{1} << 20, std::max<int64_t>(int64_t{1} << 16, count / 16));
  const int nt = static_cast<int>(std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency())));
  if (count < (int64_t{1} << 18) || nt < 2) {
    for (int64_t i = 0; i < count; ++i) out[i] = gaussian(rng);
    return;
  }
  std::vector<uint64_t> raw[2];
  raw[0].resize(2 * BLK);
  raw[1].resize(2 * BLK);
  std::vector<std::thread> pool;
  const auto join_all = [&] {
    for (auto& t : pool) t.join();
    pool.clear();
  };
  int buf = 0;
  for (int64_t i0 = 0; i0 < count; i0 += BLK, buf ^= 1) {
    const int64_t m = std::min(BLK, count - i0);
    uint64_t* rw = raw[buf].data();
    for (int64_t i = 0; i < 2 * m; ++i) rw[i] = rng();  // overlaps the previous block's transform
    join_all();
    double* dst = out + i0;
    for (int q = 0; q < nt; ++q)
      pool.emplace_back([=] {
        const int64_t a = m * q / nt, b = m * (q + 1) / nt;
        for (int64_t i = a; i < b; ++i) {
          const double u1 = (static_cast<double>(rw[2 * i] >> 11) + 0.5) * 0x1.0p-53;
          const double u2 = (static_cast<double>(rw[2 * i + 1] >> 11) + 0.5) * 0x1.0p-53;
          dst[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
        }
      });
  }
  join_all();
}
}  // namespace

bool random_block(int cx, int64_t n, int64_t k, uint64_t seed, bool orthonormalize, double* out) {
  std::mt19937_64 rng(seed);
  // complex: (re, im) interleaved in column order == the serial draw order
  gaussian_fill(rng, n * k * (cx ? 2 : 1), out);
  if (!orthonormalize) return true;
  return cx ? mgs(reinterpret_cast<std::complex<double>*>(out), n, k) : mgs(out, n, k);
}

}  // namespace zolo
