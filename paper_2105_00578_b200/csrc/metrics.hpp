// metrics.hpp — partition quality on the device (graph.cpp:184-230).
#pragma once

#include "context.hpp"

#include <vector>

namespace spb {

struct PartitionMetrics {
    double cut = 0.0;
    double imbalance = 0.0;
    std::vector<double> part_weights;
};

// a_global: device array of all n_global part ids. Validates ids and non-empty
// parts (SP_INVALID like the reference's std::invalid_argument).
PartitionMetrics make_partition_dev(sp_context* ctx, const DevGraph& g, const int32_t* a_global,
                                    int64_t K, bool doubled);
double imbalance_of(const std::vector<double>& part_weights);
double cutsize_dev(sp_context* ctx, const DevGraph& g, const int32_t* a_global, bool doubled);

} // namespace spb
