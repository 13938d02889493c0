// Request sharding for the multi-GPU request stream (BASELINE.json north_star:
// "a stream of variable-length inference requests is partitioned across the 8
// GPUs ..., each GPU running whole requests").  Deterministic LPT (longest
// processing time first) on the BERT-large flop cost of a request.
#include <algorithm>
#include <numeric>
#include <vector>

#include "internal.h"

extern "C" int64_t nimble_request_cost(int64_t L) {
    // 24 layers x (24 L d^2 + 4 L^2 d) with d = 1024: dense + attention flops
    const int64_t d = 1024;
    return 24 * (24 * L * d * d + 4 * L * L * d);
}

extern "C" int nimble_partition_lpt(const int64_t *lens, int64_t R, int32_t G, int32_t *owner) {
    using namespace nimble;
    if (R < 0 || G < 1) return fail(NIMBLE_E_EXTENT, "nimble_partition_lpt: need R >= 0 and G >= 1");
    if (R > 0 && (!lens || !owner)) return fail(NIMBLE_E_NULL, "nimble_partition_lpt: NULL array");
    for (int64_t i = 0; i < R; ++i)
        if (lens[i] < 1 || lens[i] > kMaxExtent) return fail(NIMBLE_E_EXTENT, "nimble_partition_lpt: length < 1");
    std::vector<int64_t> order(R);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return nimble_request_cost(lens[a]) > nimble_request_cost(lens[b]);   // ties keep id order
    });
    std::vector<int64_t> load(G, 0);
    for (int64_t id : order) {
        const int32_t g = static_cast<int32_t>(std::min_element(load.begin(), load.end()) - load.begin());
        owner[id] = g;                       // min_element returns the lowest rank on ties
        load[g] += nimble_request_cost(lens[id]);
    }
    clear_error();
    return NIMBLE_OK;
}
