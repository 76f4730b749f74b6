#pragma once
// Drop-in for proj/include/anisocg/cost_model.hpp: the paper's per-point cost
// tables (Tables 1-2) used by the reference's bench reporting. Implementation:
// paper_1302_7193_b200/csrc/host/cost_model.cpp.
#include <cstdint>
#include <string_view>

namespace anisocg {

enum class Kernel { spmv, prec, blas, interleaved_spmv, interleaved_prec, pcg_total, interleaved_total };
enum class CacheAssumption { none, matrix_cached, columns_cached };
enum class BlasOp { scal, axpy, dot, nrm2 };

struct CostReport {
    int flops = 0;     ///< floating-point operations per grid point
    int mem_refs = 0;  ///< memory references per grid point
};

struct ThroughputEstimate {
    double flop_rate = 0.0;  ///< flop/s
    double bandwidth = 0.0;  ///< bytes/s
};

CostReport cost_model(Kernel kernel, CacheAssumption cache);
CostReport blas_op_cost(BlasOp op);
/// flops * points / seconds and mem_refs * points * scalar_bytes / seconds
ThroughputEstimate throughput_estimate(const CostReport& report, std::int64_t grid_points,
                                       double seconds, int scalar_bytes = 8);

std::string_view to_string(Kernel kernel);
std::string_view to_string(CacheAssumption cache);
std::string_view to_string(BlasOp op);

}  // namespace anisocg
