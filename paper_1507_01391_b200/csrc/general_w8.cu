// general_w8.cu -- general-sort kernels for 8-row machines (4 per warp).
#include "general_sub.inc"

namespace dmmhost {

dmm_status launch_general_w8(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 8: return launch_sub_shape<8, 8>(mode, pk2, ext, a);
        case 16: return launch_sub_shape<8, 16>(mode, pk2, ext, a);
        case 32: return launch_sub_shape<8, 32>(mode, pk2, ext, a);
        case 64: return launch_sub_shape<8, 64>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
