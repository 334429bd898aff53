// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_spatial.hpp header).
//
// Batch layer restated from proj/core/include/vecdyn/batch.hpp:15-165:
// StateBatch (column-major N x n == SoA planes), random_states
// (mt19937_64, U[-π, π], per-state per-joint draw order q, qd, [qdd], [tau]),
// and batch_eval (row 0 on the caller, then static contiguous chunks on
// std::thread; bitwise equal to serial evaluation).
#pragma once

#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "orc_algo.hpp"

namespace orc {

struct StateBatch {
  int N = 0, n = 0;
  std::vector<double> q, qd, qdd, tau;  // column-major N x n (element (i,j) at j*N + i)
  double at(const std::vector<double>& a, int i, int j) const { return a[(size_t)j * N + i]; }
  std::vector<double> row(const std::vector<double>& a, int i) const {
    std::vector<double> r((size_t)n);
    for (int j = 0; j < n; ++j) r[(size_t)j] = a[(size_t)j * N + i];
    return r;
  }
};

// batch.hpp:48-75
inline StateBatch random_states(const Model& m, int count, uint64_t seed, bool with_qdd = true,
                                bool with_tau = false) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(-M_PI, M_PI);
  StateBatch b;
  b.N = count;
  b.n = m.dof();
  const size_t sz = (size_t)count * b.n;
  b.q.resize(sz);
  b.qd.resize(sz);
  if (with_qdd) b.qdd.resize(sz);
  if (with_tau) b.tau.resize(sz);
  for (int i = 0; i < count; ++i)
    for (int j = 0; j < b.n; ++j) {
      const size_t k = (size_t)j * count + i;
      b.q[k] = dist(rng);
      b.qd[k] = dist(rng);
      if (with_qdd) b.qdd[k] = dist(rng);
      if (with_tau) b.tau[k] = dist(rng);
    }
  return b;
}

// batch.hpp:82-125.  fn(i) evaluates row i and writes its own outputs.
template <class Fn>
void batch_eval(int count, Fn&& fn, int workers = 0) {
  if (count == 0) return;
  if (workers <= 0) workers = (int)std::thread::hardware_concurrency();
  workers = std::max(1, std::min(workers, count));
  fn(0);
  if (workers == 1 || count == 1) {
    for (int i = 1; i < count; ++i) fn(i);
    return;
  }
  const int rest = count - 1;
  const int chunk = (rest + workers - 1) / workers;
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w) {
    const int b = 1 + w * chunk, e = std::min(count, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&fn, b, e] {
      for (int i = b; i < e; ++i) fn(i);
    });
  }
  for (std::thread& t : pool) t.join();
}

}  // namespace orc
