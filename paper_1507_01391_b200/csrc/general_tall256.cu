// general_tall256.cu -- general-sort kernels for 256-row machines (one per CTA of 8 warps).
#include "general_tall.inc"

namespace dmmhost {

dmm_status launch_general_tall256(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 16: return launch_tall_shape<256, 16>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
