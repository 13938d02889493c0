// Internal host-side declarations shared by the libnimble translation units.
#pragma once
#include <cstdint>
#include <string>

#include "../../../include/nimble.h"

namespace nimble {

constexpr int64_t kMaxExtent = 2147483647LL;
constexpr int kNumSMs = 148;          // B200: 2 dies x 74 SMs

// thread-local error text (nimble_last_error)
int fail(int status, const std::string &msg);
void clear_error();
void record_dispatch(const nimble_dispatch &d);

// shape functions (shape.cc)
bool extent_ok(int64_t d);

// dispatch (dispatch.cc) — DISPATCH.md
int variant_limit();
int dispatch_simt8(int64_t M, int64_t N, nimble_dispatch *d);
int dispatch_umma_t(int64_t batch, int64_t M_tokens, int64_t N_rows, int64_t K, nimble_dispatch *d,
                    int32_t tile_t = 0, int32_t split_max = 8);
// bf16 dense: the tuned schedule registered for (N, K) (nimble_set_dense_schedule), if any
void dense_schedule(int64_t N, int64_t K, int32_t *tile_t, int32_t *split_max);
// bf16 dense: family 4 (weight streaming, M <= 128, no tuned schedule) or families 1 / 3
int dispatch_dense_bf16(int64_t M, int64_t N, int64_t K, nimble_dispatch *d);
int dispatch_umma_ws(int64_t M, int64_t N, int64_t K, nimble_dispatch *d);
int dispatch_umma_d(int64_t batch, int64_t M, int64_t N, int64_t K, nimble_dispatch *d);

}  // namespace nimble
