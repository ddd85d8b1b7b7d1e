// development: host symbolic pipeline (nd_order, block_symbolic, factor_plan) on a pattern file,
// timed on the CPU; prints the factor plan's size split by level width.
// pattern file: int64 n, int64 nnz, int64 rp[n+1], int64 ci[nnz] (union pattern, full, sorted)
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../paper_1701_08935_b200/csrc/host.hpp"

int main(int argc, char** argv) {
  FILE* f = std::fopen(argv[1], "rb");
  int64_t n, nnz;
  if (std::fread(&n, 8, 1, f) != 1 || std::fread(&nnz, 8, 1, f) != 1) return 1;
  std::vector<int64_t> rp(n + 1), ci(nnz);
  if (std::fread(rp.data(), 8, n + 1, f) != static_cast<size_t>(n + 1)) return 1;
  if (std::fread(ci.data(), 8, nnz, f) != static_cast<size_t>(nnz)) return 1;
  std::fclose(f);
  using clk = std::chrono::steady_clock;
  auto t0 = clk::now();
  std::vector<std::vector<int64_t>> nodes;
  zolo::nd_order(n, rp.data(), ci.data(), 192, nodes);
  auto t1 = clk::now();
  zolo::BlockStructure bs;
  zolo::block_symbolic(n, rp.data(), ci.data(), nodes, 32, bs);
  auto t2 = clk::now();
  zolo::FactorPlan plan;
  zolo::factor_plan(bs, plan);
  auto t3 = clk::now();
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  int64_t single = 0, multi = 0;
  for (size_t l = 0; l + 1 < plan.lvl_ptr.size(); ++l) {
    int64_t c = 0;
    for (int t = plan.tgt_ptr[l]; t < plan.tgt_ptr[l + 1]; ++t) c += plan.tgt[2 * t + 3] - plan.tgt[2 * t + 1];
    (plan.lvl_ptr[l + 1] - plan.lvl_ptr[l] == 1 ? single : multi) += c;
  }
  // canonical hash: per level, targets sorted by (kind, id), each with its ordered contributions
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  for (size_t l = 0; l + 1 < plan.lvl_ptr.size(); ++l) {
    std::vector<int> ts;
    for (int t = plan.tgt_ptr[l]; t < plan.tgt_ptr[l + 1]; ++t) ts.push_back(t);
    std::sort(ts.begin(), ts.end(), [&](int a, int b) {
      return static_cast<unsigned>(plan.tgt[2 * a]) < static_cast<unsigned>(plan.tgt[2 * b]);  // (kind, id) packed
    });
    for (int t : ts) {
      mix(static_cast<unsigned>(plan.tgt[2 * t]) >> 30);
      mix(plan.tgt[2 * t] & 0x3fffffff);
      for (int q = plan.tgt[2 * t + 1]; q < plan.tgt[2 * t + 3]; ++q) mix(plan.con[2 * q]), mix(plan.con[2 * q + 1]);
    }
    for (int q = plan.pan_ptr[l]; q < plan.pan_ptr[l + 1]; ++q) mix(plan.pan[2 * q]), mix(plan.pan[2 * q + 1]);
  }
  std::printf("plan hash %016llx\n", static_cast<unsigned long long>(h));
  std::printf("nb %lld tiles %lld levels %zu: nd %.1f ms, block_symbolic %.1f ms, factor_plan %.1f ms; "
              "contributions %lld (single-column levels %lld, multi %lld), targets %zu\n",
              static_cast<long long>(bs.nb), static_cast<long long>(bs.ntiles), plan.lvl_ptr.size() - 1, ms(t0, t1),
              ms(t1, t2), ms(t2, t3), static_cast<long long>(plan.contributions), static_cast<long long>(single),
              static_cast<long long>(multi), plan.tgt.size() / 2 - 1);
  std::printf("split targets %zu, scratch slots %lld\n", plan.cmb.size() / 3, static_cast<long long>(plan.scratch_slots));
  return 0;
}
