// WorkerPool / shard semantics (the reference's proj/tests/test_parallel.cpp
// contract) against csrc/host/parallel.cpp. Built and run by
// tests/test_pool.py; prints "ok <checks>" or the first failure.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "parallel.hpp"

static int checks = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    ++checks;                                                          \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      std::exit(1);                                                    \
    }                                                                  \
  } while (0)

template <typename E, typename F>
static std::string throws(F&& f) {
  try {
    f();
  } catch (const E& e) {
    return std::string("threw:") + e.what();
  } catch (...) {
    return "wrong type";
  }
  return "no throw";
}

int main() {
  using dopf::shard;
  using dopf::WorkerPool;
  {  // exact division
    const auto p = shard(50, 5);
    EXPECT(p.worker_count() == 5);
    for (int w = 0; w < 5; ++w) EXPECT(p.shard_size(w) == 10);
    EXPECT(p.ranges.front() == std::make_pair(0, 10) && p.ranges.back() == std::make_pair(40, 50));
  }
  {  // remainder to the first workers
    const auto p = shard(7, 3);
    EXPECT(p.shard_size(0) == 3 && p.shard_size(1) == 2 && p.shard_size(2) == 2);
  }
  {  // more workers than work
    const auto p = shard(3, 8);
    int ones = 0, idle = 0;
    for (int w = 0; w < 8; ++w) {
      ones += p.shard_size(w) == 1;
      idle += p.shard_size(w) == 0;
    }
    EXPECT(p.worker_count() == 8 && ones == 3 && idle == 5);
  }
  for (int count : {0, 1, 7, 64})  // contiguous partition
    for (int workers : {1, 2, 3, 16}) {
      int at = 0;
      for (const auto& r : shard(count, workers).ranges) {
        EXPECT(r.first == at && r.second >= r.first);
        at = r.second;
      }
      EXPECT(at == count);
    }
  for (int workers : {1, 2, 8}) {  // exactly once, repeated passes on one pool
    WorkerPool pool(workers);
    for (int pass = 0; pass < 50; ++pass) {
      std::vector<std::atomic<int>> hits(123);
      for (auto& h : hits) h = 0;
      pool.run(123, [&](int s) { ++hits[s]; });
      for (auto& h : hits) EXPECT(h.load() == 1);
    }
  }
  {  // bitwise identical outputs for any worker count
    auto body = [](int s) {
      double v = 1.0 + s;
      for (int k = 0; k < 50; ++k) v = std::sin(v) * 1.7 + std::sqrt(v + 2.0);
      return v;
    };
    std::vector<double> ref(37);
    WorkerPool one(1);
    one.run(37, [&](int s) { ref[s] = body(s); });
    for (int workers : {4, 16}) {
      std::vector<double> out(37);
      WorkerPool pool(workers);
      pool.run(37, [&](int s) { out[s] = body(s); });
      for (int s = 0; s < 37; ++s) EXPECT(out[s] == ref[s]);
    }
  }
  {  // a throwing body names the (lowest) failing subsystem; the pool stays usable
    WorkerPool pool(3);
    for (int rep = 0; rep < 20; ++rep) {
      const std::string r = throws<std::runtime_error>([&] {
        pool.run(9, [&](int s) {
          if (s == 5 || s == 8) throw std::runtime_error("boom");
        });
      });
      EXPECT(r.find("subsystem 5") != std::string::npos && r.find("boom") != std::string::npos);
    }
    std::vector<std::atomic<int>> hits(4);
    for (auto& h : hits) h = 0;
    pool.run(4, [&](int s) { ++hits[s]; });
    for (auto& h : hits) EXPECT(h.load() == 1);
  }
  EXPECT(throws<std::invalid_argument>([] { WorkerPool p(0); }).rfind("threw:", 0) == 0);
  EXPECT(throws<std::invalid_argument>([] { shard(5, 0); }).rfind("threw:", 0) == 0);
  {  // a plan with more shards than workers is rejected
    WorkerPool pool(2);
    EXPECT(throws<std::invalid_argument>([&] { pool.run(shard(10, 3), [](int) {}); }).rfind("threw:", 0) == 0);
  }
  std::printf("ok %d\n", checks);
  return 0;
}
