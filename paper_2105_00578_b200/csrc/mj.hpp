// mj.hpp — device multi-jagged partitioner (partitioner.cpp:43-170).
#pragma once

#include "common.cuh"

#include <vector>

namespace spb {

// MjPlan (partitioner.hpp:26-34): leaves = node target, dim = cut dimension
// (-1 for leaves), kids in section order.
struct MjPlanNode {
    int64_t leaves = 1;
    int dim = -1;
    std::vector<MjPlanNode> kids;
    int64_t leaf_count() const;
};

MjPlanNode mj_plan(int64_t num_parts, int dims);

// coords: n x dims view on the device (point i, coordinate c = coords.at(i, c)).
// weights_dev: n positive weights (ignored when unit_weights). Writes part ids
// in [0, K) to assignment_dev (device, n).
void mj_partition_dev(int64_t n, int dims, const View& coords, const double* weights_dev,
                      bool unit_weights, int64_t num_parts, int32_t* assignment_dev, cudaStream_t s);

} // namespace spb
