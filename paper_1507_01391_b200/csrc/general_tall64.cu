// general_tall64.cu -- general-sort kernels for 64-row machines (one per CTA of 2 warps).
#include "general_tall.inc"

namespace dmmhost {

dmm_status launch_general_tall64(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 8: return launch_tall_shape<64, 8>(mode, pk2, ext, a);
        case 16: return launch_tall_shape<64, 16>(mode, pk2, ext, a);
        case 32: return launch_tall_shape<64, 32>(mode, pk2, ext, a);
        case 64: return launch_tall_shape<64, 64>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
