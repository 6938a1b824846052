// general_m128.cu -- instantiations of the general-sort kernel for 32 x 128 machines
// (w <= m: integer_sort_general / partition_general reduce to the leaf, cfg3's sort).
#include "general_kernel.cuh"

namespace dmmhost {

dmm_status launch_general_m128(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    switch (mode) {
        case dmmdev::kModePartition:
            return launch_general<128, 2, false, dmmdev::kModePartition>(a);
        case dmmdev::kModeIntegerSort:
            return pk2 ? launch_general<128, 2, false, dmmdev::kModeIntegerSort>(a)
                       : launch_general<128, 1, false, dmmdev::kModeIntegerSort>(a);
        default:
            set_error("sort_wide_any is built for m = 32, 64");
            return DMM_UNSUPPORTED_SHAPE;
    }
}

}  // namespace dmmhost
