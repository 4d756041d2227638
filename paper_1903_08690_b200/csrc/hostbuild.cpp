// hostbuild.cpp — native host helpers for index construction and the seeded
// BASELINE-config data generator (libhsbuild.so, plain C ABI, OpenMP).
//
// Index construction is not the graded hot path, but
// the reference's Python loops make it the wall-clock bottleneck at the
// BASELINE sizes (cache_sort took 62 s at N=1e5, sparse.py:138-163).  These
// helpers restate the integer parts exactly:
//   hsb_cache_sort      cache_sort + _refine_equal_runs (sparse.py:106-163):
//                       stable sort of points by their activity pattern over
//                       the dims ranked (nnz desc, dim asc), descending
//                       lexicographically.  Equivalent comparator: compare the
//                       ascending rank lists; the first differing rank that is
//                       smaller wins; a proper prefix sorts after its extension.
//   hsb_top_t_thresholds _top_t_thresholds (sparse.py:66-80): t-th largest |v|.
// and generate synthetic hybrid data with the BASELINE laws.
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---- counter-based RNG (splitmix64 over a (seed, stream, counter) key) ----
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct Rng {
  uint64_t s;
  Rng(uint64_t seed, uint64_t stream) : s(mix64(seed * 0x100000001B3ULL ^ mix64(stream + 1))) {}
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }  // (0,1)
  double normal() {
    const double u1 = uniform(), u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
  // Poisson by inversion for small means, normal approximation above 500
  int64_t poisson(double mean) {
    if (mean <= 0) return 0;
    if (mean > 500) {
      const double x = std::floor(mean + std::sqrt(mean) * normal() + 0.5);
      return x < 0 ? 0 : (int64_t)x;
    }
    const double L = std::exp(-mean);
    int64_t k = 0;
    double p = 1.0;
    do {
      ++k;
      p *= uniform();
    } while (p > L);
    return k - 1;
  }
};

// ---- seeded bijection of [0, d): 4-round Feistel on 2w bits + cycle walking ----
struct Feistel {
  uint64_t d;
  int half;
  uint64_t mask;
  uint64_t keys[4];
  Feistel(uint64_t d_, uint64_t seed) : d(d_) {
    int bits = 2;
    while ((1ULL << bits) < d) bits += 2;
    half = bits / 2;
    mask = (1ULL << half) - 1;
    for (int r = 0; r < 4; ++r) keys[r] = mix64(seed ^ (0xA5A5A5A5ULL + r));
  }
  uint64_t once(uint64_t x) const {
    uint64_t L = x >> half, R = x & mask;
    for (int r = 0; r < 4; ++r) {
      const uint64_t F = mix64(R ^ keys[r]) & mask;
      const uint64_t nL = R;
      R = L ^ F;
      L = nL;
    }
    return (L << half) | R;
  }
  uint64_t operator()(uint64_t x) const {
    uint64_t y = once(x);
    while (y >= d) y = once(y);
    return y;
  }
};

}  // namespace

extern "C" {

// Generate n rows of the BASELINE law.
//   nnz per row ~ Poisson(mean_nnz), that many DISTINCT dims drawn from
//   Zipf(s) over ranks 1..d_sparse (inverse CDF), mapped through a seeded
//   bijection shared by data and queries (perm_seed);
//   value_law 0: |N(0,1)|, 1: lognormal(0,1);  dense: N(0,1).
//   Each row scaled by 1/||[x_s, x_d]|| computed in f64, stored f32;
//   dense_fp16 != 0 rounds the normalised dense part to fp16 (cfg 5).
// Two-call protocol: pass indices == NULL to get row counts in indptr
// (indptr[n] = total nnz), then call again with buffers.
int hsb_gen_hybrid(int64_t n, int64_t d_sparse, int64_t d_dense, double mean_nnz,
                   double zipf_s, int value_law, uint64_t seed, uint64_t perm_seed,
                   int dense_fp16, int64_t* indptr, int32_t* indices, float* data,
                   float* dense) {
  if (n < 0 || d_sparse < 0 || d_dense < 0) return 1;
  const uint64_t cnt_stream = 0x1000000000ULL;
  if (!indices) {
    indptr[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      Rng r(seed, cnt_stream + (uint64_t)i);
      int64_t k = d_sparse ? r.poisson(mean_nnz) : 0;
      if (k > d_sparse) k = d_sparse;
      indptr[i + 1] = k;
    }
    for (int64_t i = 0; i < n; ++i) indptr[i + 1] += indptr[i];
    return 0;
  }
  // Zipf CDF over ranks (truncated at d_sparse); for huge d a continuous tail
  const int64_t table_n = std::min<int64_t>(d_sparse, 1 << 24);
  std::vector<double> cdf(std::max<int64_t>(table_n, 1));
  double acc = 0.0;
  for (int64_t r = 0; r < table_n; ++r) {
    acc += std::pow((double)(r + 1), -zipf_s);
    cdf[r] = acc;
  }
  double tail = 0.0;  // mass of ranks beyond the table (integral approximation)
  if (d_sparse > table_n) {
    const double a = (double)table_n + 0.5, b = (double)d_sparse + 0.5;
    tail = (std::pow(a, 1.0 - zipf_s) - std::pow(b, 1.0 - zipf_s)) / (zipf_s - 1.0);
  }
  const double total = acc + tail;
  Feistel perm((uint64_t)std::max<int64_t>(d_sparse, 1), perm_seed);

#pragma omp parallel
  {
    std::vector<int64_t> ranks;
    std::vector<double> vals;
    std::vector<std::pair<int64_t, double>> row;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
      Rng r(seed, (uint64_t)i);
      const int64_t k = indptr[i + 1] - indptr[i];
      ranks.clear();
      while ((int64_t)ranks.size() < k) {
        const double u = r.uniform() * total;
        int64_t rank;
        if (u < acc || tail == 0.0) {
          rank = std::lower_bound(cdf.begin(), cdf.begin() + table_n, u) - cdf.begin();
          if (rank >= table_n) rank = table_n - 1;
        } else {
          // invert the continuous tail
          const double a = (double)table_n + 0.5;
          const double rem = u - acc;
          const double x = std::pow(std::pow(a, 1.0 - zipf_s) - rem * (zipf_s - 1.0),
                                    1.0 / (1.0 - zipf_s));
          rank = (int64_t)std::floor(x - 0.5);
          if (rank < table_n) rank = table_n;
          if (rank >= d_sparse) rank = d_sparse - 1;
        }
        if (std::find(ranks.begin(), ranks.end(), rank) == ranks.end()) ranks.push_back(rank);
      }
      row.clear();
      double ss = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        double v;
        if (value_law == 1) v = std::exp(r.normal());
        else v = std::fabs(r.normal());
        if (v == 0.0) v = 1e-30;
        row.emplace_back((int64_t)perm((uint64_t)ranks[j]), v);
        ss += v * v;
      }
      std::vector<double> dv(d_dense);
      for (int64_t j = 0; j < d_dense; ++j) {
        dv[j] = r.normal();
        ss += dv[j] * dv[j];
      }
      const double inv = ss > 0 ? 1.0 / std::sqrt(ss) : 1.0;
      std::sort(row.begin(), row.end());
      const int64_t o = indptr[i];
      for (int64_t j = 0; j < k; ++j) {
        indices[o + j] = (int32_t)row[j].first;
        float f = (float)(row[j].second * inv);
        if (f == 0.0f) f = 1e-38f;
        data[o + j] = f;
      }
      for (int64_t j = 0; j < d_dense; ++j) {
        float f = (float)(dv[j] * inv);
        if (dense_fp16) {
          // round-to-nearest-even to fp16 then back
          _Float16 h = (_Float16)f;
          f = (float)h;
        }
        dense[i * d_dense + j] = f;
      }
    }
  }
  return 0;
}

// Stable layout sort.  rows: CSR (indptr over n points) of the ranks of each
// point's active dims, each row sorted ascending.  order[slot] = point id.
int hsb_cache_sort(int64_t n, const int64_t* indptr, const int32_t* ranks, int64_t* order) {
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  auto cmp = [&](int64_t a, int64_t b) {
    int64_t ia = indptr[a], ea = indptr[a + 1];
    int64_t ib = indptr[b], eb = indptr[b + 1];
    for (;;) {
      const bool da = ia == ea, db = ib == eb;
      if (da || db) return !da && db;  // a longer (has an extra rank) -> a first
      const int32_t ra = ranks[ia], rb = ranks[ib];
      if (ra != rb) return ra < rb;
      ++ia;
      ++ib;
    }
  };
  std::stable_sort(idx.begin(), idx.end(), cmp);
  std::memcpy(order, idx.data(), sizeof(int64_t) * n);
  return 0;
}

// eta[j] = t-th largest |v| in column j when nnz_j > t, else 0 (CSC input).
int hsb_top_t_thresholds(int64_t d, const int64_t* indptr, const float* data, int64_t t,
                         double* eta) {
#pragma omp parallel
  {
    std::vector<double> col;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t j = 0; j < d; ++j) {
      const int64_t lo = indptr[j], hi = indptr[j + 1], m = hi - lo;
      if (t == 0) {
        eta[j] = INFINITY;
        continue;
      }
      if (m <= t) {
        eta[j] = 0.0;
        continue;
      }
      col.resize(m);
      for (int64_t i = 0; i < m; ++i) col[i] = std::fabs((double)data[lo + i]);
      std::nth_element(col.begin(), col.begin() + (m - t), col.end());
      eta[j] = col[m - t];
    }
  }
  return 0;
}


// ---------------------------------------------------------------------------
// prune_split (sparse.py:83-103): per-column thresholds from a CSR matrix and
// the three-way split.  Thresholds: eta[j] = t-th largest |v| in column j
// when nnz_j > t (np.partition semantics), 0 otherwise; t == 0 -> +inf.
// ---------------------------------------------------------------------------
int hsb_top_t_thresholds_csr(int64_t n, int64_t d, const int64_t* indptr,
                             const int32_t* indices, const float* data, int64_t t,
                             double* eta) {
  if (t == 0) {
    for (int64_t j = 0; j < d; ++j) eta[j] = INFINITY;
    return 0;
  }
  std::vector<int64_t> cnt(d + 1, 0);
  const int64_t nnz = indptr[n];
  for (int64_t e = 0; e < nnz; ++e) cnt[indices[e] + 1]++;
  for (int64_t j = 0; j < d; ++j) cnt[j + 1] += cnt[j];
  std::vector<float> vals(nnz);
  std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
  for (int64_t e = 0; e < nnz; ++e) vals[cur[indices[e]]++] = std::fabs(data[e]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t j = 0; j < d; ++j) {
    const int64_t lo = cnt[j], m = cnt[j + 1] - lo;
    if (m <= t) {
      eta[j] = 0.0;
      continue;
    }
    std::nth_element(vals.begin() + lo, vals.begin() + lo + (m - t), vals.begin() + lo + m);
    eta[j] = (double)vals[lo + (m - t)];
  }
  return 0;
}

// Two-call protocol: with d_indices == NULL fills d_indptr / r_indptr
// (cumulative); then fills both parts.  Entries with v == 0 are dropped
// (eliminate_zeros, sparse.py:99-101).
int hsb_prune_split(int64_t n, const int64_t* indptr, const int32_t* indices, const float* data,
                    const double* eta, const double* eps, int64_t* d_indptr, int32_t* d_indices,
                    float* d_data, int64_t* r_indptr, int32_t* r_indices, float* r_data) {
  auto cls = [&](int64_t e) -> int {  // 0 data, 1 residual, 2 discard
    const float v = data[e];
    if (v == 0.0f) return 2;
    const double a = std::fabs((double)v);
    const int32_t j = indices[e];
    if (a >= eta[j]) return 0;
    if (a >= eps[j]) return 1;
    return 2;
  };
  if (!d_indices) {
    d_indptr[0] = 0;
    r_indptr[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      int64_t a = 0, b = 0;
      for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
        const int c = cls(e);
        a += c == 0;
        b += c == 1;
      }
      d_indptr[i + 1] = a;
      r_indptr[i + 1] = b;
    }
    for (int64_t i = 0; i < n; ++i) {
      d_indptr[i + 1] += d_indptr[i];
      r_indptr[i + 1] += r_indptr[i];
    }
    return 0;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = d_indptr[i], b = r_indptr[i];
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      const int c = cls(e);
      if (c == 0) {
        d_indices[a] = indices[e];
        d_data[a++] = data[e];
      } else if (c == 1) {
        r_indices[b] = indices[e];
        r_data[b++] = data[e];
      }
    }
  }
  return 0;
}

// Per-row ascending ranks (rank_of maps dim -> rank) for cache_sort.
int hsb_rank_rows(int64_t n, const int64_t* indptr, const int32_t* indices,
                  const int32_t* rank_of, int32_t* ranks) {
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) ranks[e] = rank_of[indices[e]];
    std::sort(ranks + indptr[i], ranks + indptr[i + 1]);
  }
  return 0;
}

// build_inverted (sparse.py:219-235): counts per column, then fill the
// posting lists (slot ids ascending within each list).
int hsb_inverted_counts(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                        const float* data, int64_t* counts) {
  for (int64_t j = 0; j < d; ++j) counts[j] = 0;
  const int64_t nnz = indptr[n];
  for (int64_t e = 0; e < nnz; ++e)
    if (data[e] != 0.0f) counts[indices[e]]++;
  return 0;
}

int hsb_inverted_fill(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                      const float* data, const int64_t* pos, const int64_t* colptr,
                      uint32_t* ids, float* w) {
  std::vector<int64_t> cur(colptr, colptr + d);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      if (data[e] == 0.0f) continue;
      const int64_t at = cur[indices[e]]++;
      ids[at] = (uint32_t)pos[i];
      w[at] = data[e];
    }
#pragma omp parallel
  {
    std::vector<std::pair<uint32_t, float>> tmp;
#pragma omp for schedule(dynamic, 4096)
    for (int64_t j = 0; j < d; ++j) {
      const int64_t lo = colptr[j], hi = colptr[j + 1];
      if (hi - lo < 2) continue;
      tmp.resize(hi - lo);
      for (int64_t k = lo; k < hi; ++k) tmp[k - lo] = {ids[k], w[k]};
      std::sort(tmp.begin(), tmp.end(),
                [](const std::pair<uint32_t, float>& a, const std::pair<uint32_t, float>& b) {
                  return a.first < b.first;
                });
      for (int64_t k = lo; k < hi; ++k) {
        ids[k] = tmp[k - lo].first;
        w[k] = tmp[k - lo].second;
      }
    }
  }
  return 0;
}

// pq_encode (dense.py:138-153) for subspaces of width <= 2, reproducing
// numpy's arithmetic: |x|^2 summed from 0, the 2-wide BLAS product
// fma(x1, c1, x0*c0), d2 = (|x|^2 - 2*dot) + |c|^2, first minimum wins.
// Returns 1 if a subspace is wider than 2 (caller falls back).
int hsb_pq_encode(int64_t n, int64_t d, const double* x, int32_t K, const int64_t* subdims,
                  const float* centers, int32_t l, uint8_t* codes) {
  std::vector<int64_t> off(K), coff(K);
  int64_t o = 0, co = 0;
  for (int32_t k = 0; k < K; ++k) {
    if (subdims[k] > 2 || subdims[k] < 1) return 1;
    off[k] = o;
    coff[k] = co;
    o += subdims[k];
    co += subdims[k] * l;
  }
  std::vector<double> csq((size_t)K * l);
  for (int32_t k = 0; k < K; ++k)
    for (int32_t c = 0; c < l; ++c) {
      const float* cc = centers + coff[k] + (int64_t)c * subdims[k];
      double s = 0.0;
      for (int64_t t = 0; t < subdims[k]; ++t) {
        const double v = (double)cc[t];
        s = s + v * v;
      }
      csq[(size_t)k * l + c] = s;
    }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* xi = x + i * d;
    for (int32_t k = 0; k < K; ++k) {
      const double* s = xi + off[k];
      const float* cb = centers + coff[k];
      int best = 0;
      double bd = 0.0;
      if (subdims[k] == 2) {
        const double sq = (0.0 + s[0] * s[0]) + s[1] * s[1];
        for (int32_t c = 0; c < l; ++c) {
          const double c0 = cb[2 * c], c1 = cb[2 * c + 1];
          const double dot = std::fma(s[1], c1, s[0] * c0);
          const double d2 = (sq - 2.0 * dot) + csq[(size_t)k * l + c];
          if (c == 0 || d2 < bd) {
            bd = d2;
            best = c;
          }
        }
      } else {
        const double sq = 0.0 + s[0] * s[0];
        for (int32_t c = 0; c < l; ++c) {
          const double dot = s[0] * (double)cb[c];
          const double d2 = (sq - 2.0 * dot) + csq[(size_t)k * l + c];
          if (c == 0 || d2 < bd) {
            bd = d2;
            best = c;
          }
        }
      }
      codes[i * K + k] = (uint8_t)best;
    }
  }
  return 0;
}

// Scalar-quantised dense residual (pipeline.py:158-160, dense.py:381-390):
// r = vec[order[i]] - center(code) in f64; per-dim lo/hi; step = (hi-lo)/256;
// code = clip(floor((r - lo) / (step > 0 ? step : 1)), 0, 255).
int hsb_sq_residual(int64_t n, int64_t d, const double* vec, const int64_t* order,
                    const uint8_t* codes, int32_t K, const int64_t* subdims, const float* centers,
                    int32_t l, float* lo_out, float* step_out, uint8_t* sq) {
  std::vector<int64_t> dimk(d), dimt(d), coff(K);
  int64_t o = 0, co = 0;
  for (int32_t k = 0; k < K; ++k) {
    coff[k] = co;
    for (int64_t t = 0; t < subdims[k]; ++t) {
      dimk[o] = k;
      dimt[o] = t;
      ++o;
    }
    co += subdims[k] * l;
  }
  auto resid = [&](int64_t i, int64_t j) -> double {
    const int64_t k = dimk[j];
    const int c = codes[i * K + k];
    return vec[order[i] * d + j] - (double)centers[coff[k] + (int64_t)c * subdims[k] + dimt[j]];
  };
  std::vector<double> lo(d, INFINITY), hi(d, -INFINITY);
#pragma omp parallel
  {
    std::vector<double> tlo(d, INFINITY), thi(d, -INFINITY);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < d; ++j) {
        const double r = resid(i, j);
        if (r < tlo[j]) tlo[j] = r;
        if (r > thi[j]) thi[j] = r;
      }
#pragma omp critical
    for (int64_t j = 0; j < d; ++j) {
      if (tlo[j] < lo[j]) lo[j] = tlo[j];
      if (thi[j] > hi[j]) hi[j] = thi[j];
    }
  }
  std::vector<double> step(d), safe(d);
  for (int64_t j = 0; j < d; ++j) {
    if (n == 0) lo[j] = hi[j] = 0.0;
    step[j] = (hi[j] - lo[j]) / 256.0;
    safe[j] = step[j] > 0 ? step[j] : 1.0;
    lo_out[j] = (float)lo[j];
    step_out[j] = (float)step[j];
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < d; ++j) {
      double q = std::floor((resid(i, j) - lo[j]) / safe[j]);
      if (q < 0) q = 0;
      if (q > 255) q = 255;
      sq[i * d + j] = (uint8_t)q;
    }
  return 0;
}

int hsb_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
