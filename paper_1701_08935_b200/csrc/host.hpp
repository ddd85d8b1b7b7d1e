#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>

namespace zolo {
// status-carrying error thrown by the host setup (codes as include/zolo_b200.h)
struct DesignError : std::runtime_error {
  int code;
  DesignError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void rcm_order(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm);
int64_t bandwidth_under(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* perm);
int64_t profile_under(int64_t n, const int64_t* rp, const int64_t* ci, const int64_t* perm);
void uniform_stream(uint64_t seed, int64_t n, double* out);
bool random_block(int cx, int64_t n, int64_t k, uint64_t seed, bool orthonormalize, double* out);
void build_filter_design(const double* gaps, int r, double* out);
int choose_order(const double* gaps, double eps);
void eval_filter_scalar(const double* gaps, int r, int64_t npts, const double* x, double* g_out, double* f_out);
}  // namespace zolo
