// general_w2.cu -- general-sort kernels for 2-row machines (16 per warp).
#include "general_sub.inc"

namespace dmmhost {

dmm_status launch_general_w2(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 2: return launch_sub_shape<2, 2>(mode, pk2, ext, a);
        case 4: return launch_sub_shape<2, 4>(mode, pk2, ext, a);
        case 8: return launch_sub_shape<2, 8>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
