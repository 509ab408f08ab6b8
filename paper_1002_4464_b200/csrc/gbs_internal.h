// gbs_internal.h -- entry points shared between the translation units of libgbs.so
// (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/gbs.h"

namespace gbs {
gbs_status_t fail_msg(gbs_status_t st, const char* msg);
// Sort n distinct u64 composites in place (Step 4 machinery); ws sized by sort_u64_ws.
gbs_status_t sort_u64_inplace(unsigned long long* d, size_t n, void* ws, size_t ws_bytes, cudaStream_t st);
gbs_status_t sort_u64_ws(size_t n, size_t* bytes);
// Out-of-place u32 keys sort: in[0, n) read only, sorted result in out (E1 of the
// multi-GPU entry); ws sized by sort_keys_oop_ws.
gbs_status_t sort_keys_oop_ws(size_t n, size_t* bytes);
gbs_status_t sort_keys_oop(const uint32_t* in, uint32_t* out, size_t n, void* ws, size_t ws_bytes, cudaStream_t st);
// gbs_profile_begin() is active on this thread (the multi-GPU entry records its phases)
bool profiling();
}  // namespace gbs
