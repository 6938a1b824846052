// general_m32.cu -- instantiations of the general-sort kernel for 32 x 32 machines.
#include <cstdlib>

#include "general_kernel.cuh"

namespace dmmhost {

dmm_status launch_general_m32(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    // w = m: partition_leaf only (any starting layout); without a probe the persistent
    // TMA-pipelined kernel runs it (DMM_NO_PIPE=1 selects the one-task-per-warp kernel)
    static const bool no_pipe = getenv("DMM_NO_PIPE") && getenv("DMM_NO_PIPE")[0] == '1';
    const bool pipe = !a.probe && !no_pipe;
    switch (mode) {
        case dmmdev::kModePartition:
            if (pipe)
                return pk2 ? launch_general_pipe<32, 2, false, dmmdev::kModePartition>(a)
                           : launch_general_pipe<32, 1, false, dmmdev::kModePartition>(a);
            return pk2 ? launch_general<32, 2, false, dmmdev::kModePartition>(a) : launch_general<32, 1, false, dmmdev::kModePartition>(a);
        case dmmdev::kModeIntegerSort:
            if (pipe)
                return pk2 ? launch_general_pipe<32, 2, false, dmmdev::kModeIntegerSort>(a)
                           : launch_general_pipe<32, 1, false, dmmdev::kModeIntegerSort>(a);
            return pk2 ? launch_general<32, 2, false, dmmdev::kModeIntegerSort>(a) : launch_general<32, 1, false, dmmdev::kModeIntegerSort>(a);
        default:
            return pk2 ? launch_general<32, 2, false, dmmdev::kModeSortAny>(a) : launch_general<32, 1, false, dmmdev::kModeSortAny>(a);
    }
}

}  // namespace dmmhost
