// general_m64.cu -- instantiations of the general-sort kernel for 32 x 64 machines.
#include "general_kernel.cuh"

namespace dmmhost {

dmm_status launch_general_m64(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (partition_count_applies(64, mode, a))
        return launch_partition_count(64, mode, a);
    switch (mode) {
        case dmmdev::kModePartition:
            return pk2 ? launch_general<64, 2, false, dmmdev::kModePartition>(a) : launch_general<64, 1, false, dmmdev::kModePartition>(a);
        case dmmdev::kModeIntegerSort:
            return pk2 ? launch_general<64, 2, false, dmmdev::kModeIntegerSort>(a) : launch_general<64, 1, false, dmmdev::kModeIntegerSort>(a);
        default:
            return pk2 ? launch_general<64, 2, false, dmmdev::kModeSortAny>(a) : launch_general<64, 1, false, dmmdev::kModeSortAny>(a);
    }
}

}  // namespace dmmhost
