// permute.cu -- kernel 4: the randomized permutation (permute.hpp:545-628).
// (Placeholder entry points until the warp pipeline lands; no CPU fallback.)
#include "capi_common.h"

extern "C" {

uint64_t dmm_permute_workspace_bytes(uint32_t w, uint32_t m, uint64_t count) {
    (void)w;
    (void)m;
    return count * 312ull * 8ull;
}

dmm_status dmm_permute(const uint32_t* in, uint32_t* out, uint32_t w, uint32_t m, uint64_t count,
                       const uint64_t* seeds, uint32_t alpha, uint32_t iter_cap, dmm_permute_report* reports,
                       uint64_t* history, uint32_t* shifts, uint8_t* status, void* workspace, void* stream) {
    dmmhost::reset_launches();
    (void)in, (void)out, (void)count, (void)seeds, (void)alpha, (void)iter_cap, (void)reports, (void)history,
        (void)shifts, (void)status, (void)workspace, (void)stream;
    if (m < 2 || w % m != 0)  // permute.hpp:547-548
        return DMM_SHAPE_VIOLATION;
    if (!dmmhost::general_sort_shape_ok(w, m, false))  // permute.hpp:549-550
        return DMM_SHAPE_VIOLATION;
    dmmhost::set_error("dmm_permute: kernel not built yet");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // extern "C"
