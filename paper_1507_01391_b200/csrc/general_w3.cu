// general_w3.cu -- general-sort kernels for 3-row machines (10 per warp, 2 lanes idle): the
// reference's own odd test shape 3 x 9 (test_partition.cpp:92-108, partition_short_wide).
// Shapes that are not powers of two run the reference's leaf dispatch literally (short-wide
// skeleton), with Batcher row networks whose padding comparators are dropped.
#include "general_sub.inc"

namespace dmmhost {

dmm_status launch_general_w3(uint32_t m, int mode, bool pk2, bool ext, const GeneralArgs& a) {
    switch (m) {
        case 9: return launch_sub_shape<3, 9>(mode, pk2, ext, a);
        default: break;
    }
    set_error("no kernel compiled for this shape");
    return DMM_UNSUPPORTED_SHAPE;
}

}  // namespace dmmhost
