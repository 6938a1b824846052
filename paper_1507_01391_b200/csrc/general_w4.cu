// general_w4.cu -- general-sort kernels for 4-row machines (8 per warp).
#include "general_sub.inc"

namespace dmmhost {

dmm_status launch_general_w4(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 4: return launch_sub_shape<4, 4>(mode, pk2, ext, a);
        case 8: return launch_sub_shape<4, 8>(mode, pk2, ext, a);
        case 16: return launch_sub_shape<4, 16>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
