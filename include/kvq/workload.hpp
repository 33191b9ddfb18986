// kvq/workload.hpp — the per-head workload record of the reference (workload.hpp:68-72),
// as consumed by mse_report. The synthetic generator itself (generate / generate_step,
// workload.hpp:74-200) is host-side test-data code outside the B200 hot path; parity tests
// take its outputs from the reference (tests/golden) or its C restatement (oracle/).
#pragma once

#include "kvq/matrix.hpp"

namespace kvq {

struct HeadWorkload {
    DenseMatrix keys;    // tokens x head_dim
    DenseMatrix values;  // tokens x head_dim
    DenseMatrix query;   // 1 x head_dim
};

}  // namespace kvq
