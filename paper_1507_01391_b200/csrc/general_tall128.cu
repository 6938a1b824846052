// general_tall128.cu -- general-sort kernels for 128-row machines (one per CTA of 4 warps).
#include "general_tall.inc"

namespace dmmhost {

dmm_status launch_general_tall128(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 32: return launch_tall_shape<128, 32>(mode, pk2, ext, a);
        case 64: return launch_tall_shape<128, 64>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
