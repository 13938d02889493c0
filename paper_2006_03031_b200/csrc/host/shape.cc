// Shape functions (Nimble §3.2): data-independent mode, run on
// the host ("shape functions ... on a CPU domain").
// With NIMBLE_ANY inputs they act as the compile-time type relation (§3.1).
#include "internal.h"

namespace nimble {

bool extent_ok(int64_t d) { return d == NIMBLE_ANY || (d >= 1 && d <= kMaxExtent); }

// broadcast_rel for one dimension; static pairs follow numpy broadcasting.
static int broadcast_rel(int64_t a, int64_t b, int64_t *out) {
    const bool a_any = (a == NIMBLE_ANY), b_any = (b == NIMBLE_ANY);
    if (a_any || b_any) {
        const int64_t other = a_any ? b : a;
        // (Any,Any)->Any; (Any,1)->Any; (Any,d>1)->d with a deferred runtime check
        *out = (other == NIMBLE_ANY || other == 1) ? NIMBLE_ANY : other;
        return NIMBLE_OK;
    }
    if (a == b || b == 1) { *out = a; return NIMBLE_OK; }
    if (a == 1) { *out = b; return NIMBLE_OK; }
    return NIMBLE_E_SHAPE;
}

}  // namespace nimble

using namespace nimble;

extern "C" int nimble_shape_dense(const int64_t x_shape[2], const int64_t w_shape[2], int64_t out_shape[2]) {
    if (!x_shape || !w_shape || !out_shape) return fail(NIMBLE_E_NULL, "nimble_shape_dense: NULL shape array");
    for (int i = 0; i < 2; ++i)
        if (!extent_ok(x_shape[i]) || !extent_ok(w_shape[i]))
            return fail(NIMBLE_E_EXTENT, "nimble_shape_dense: extent must be >= 1 or NIMBLE_ANY");
    const int64_t kx = x_shape[1], kw = w_shape[1];
    if (kx != NIMBLE_ANY && kw != NIMBLE_ANY && kx != kw)
        return fail(NIMBLE_E_SHAPE, "nimble_shape_dense: K mismatch x[1]=" + std::to_string(kx) +
                                        " W[1]=" + std::to_string(kw));
    out_shape[0] = x_shape[0];
    out_shape[1] = w_shape[0];
    return NIMBLE_OK;
}

extern "C" int nimble_shape_bmm(const int64_t a_shape[3], const int64_t b_shape[3], int trans_b,
                                int64_t out_shape[3]) {
    if (!a_shape || !b_shape || !out_shape) return fail(NIMBLE_E_NULL, "nimble_shape_bmm: NULL shape array");
    for (int i = 0; i < 3; ++i)
        if (!extent_ok(a_shape[i]) || !extent_ok(b_shape[i]))
            return fail(NIMBLE_E_EXTENT, "nimble_shape_bmm: extent must be >= 1 or NIMBLE_ANY");
    const int64_t kb = trans_b ? b_shape[1] : b_shape[2];
    const int64_t nb = trans_b ? b_shape[2] : b_shape[1];
    if (a_shape[2] != NIMBLE_ANY && kb != NIMBLE_ANY && a_shape[2] != kb)
        return fail(NIMBLE_E_SHAPE, "nimble_shape_bmm: K mismatch");
    int64_t batch = 0;
    if (broadcast_rel(a_shape[0], b_shape[0], &batch) != NIMBLE_OK)
        return fail(NIMBLE_E_SHAPE, "nimble_shape_bmm: batch dims do not broadcast");
    out_shape[0] = batch;
    out_shape[1] = a_shape[1];
    out_shape[2] = nb;
    return NIMBLE_OK;
}
