// general_m8.cu -- instantiations of the general-sort kernel for 32 x 8 machines.
#include "general_kernel.cuh"

namespace dmmhost {

dmm_status launch_general_m8(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        if (mode == dmmdev::kModePartition)
            return pk2 ? launch_general<8, 2, true, dmmdev::kModePartition>(a) : launch_general<8, 1, true, dmmdev::kModePartition>(a);
        if (mode == dmmdev::kModeIntegerSort)
            return pk2 ? launch_general<8, 2, true, dmmdev::kModeIntegerSort>(a) : launch_general<8, 1, true, dmmdev::kModeIntegerSort>(a);
    }
    set_error("32 x 8 needs DMM_FLAG_EXT_PARTIAL_GROUPS (the reference rejects it, partition.hpp:241-244)");
    return DMM_SHAPE_VIOLATION;
}

}  // namespace dmmhost
