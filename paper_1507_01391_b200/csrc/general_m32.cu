// general_m32.cu -- instantiations of the general-sort kernel for 32 x 32 machines.
#include <cstdlib>

#include "general_kernel.cuh"

namespace dmmhost {

dmm_status launch_general_m32(int mode, bool pk2, bool ext, const GeneralArgs& a) {
    if (ext) {
        set_error("extension kernels are only built where the reference rejects the shape");
        return DMM_UNSUPPORTED_SHAPE;
    }
    if (partition_count_applies(32, mode, a))
        return launch_partition_count(32, mode, a);
    // w = m: partition_leaf only (any starting layout).  DMM_PIPE selects a persistent variant
    // (2 = L2 prefetch of the next task, 1 = TMA into a per-warp shared-memory slot); both
    // measured SLOWER than one task per warp (0, the default): 320 / 321 vs 351 G keys/s on
    // cfg1 (profiles/r02/pipeline_ab.txt) -- fewer resident warps (1) or a longer register
    // lifetime (2) cost more than the hidden load latency gains.
    static const int pipe_mode = getenv("DMM_PIPE") ? atoi(getenv("DMM_PIPE")) : 0;
    const bool pipe = !a.probe && pipe_mode != 0;
    switch (mode) {
        case dmmdev::kModePartition:
            if (pipe && pipe_mode == 1)
                return pk2 ? launch_general_pipe<32, 2, false, dmmdev::kModePartition, 1>(a)
                           : launch_general_pipe<32, 1, false, dmmdev::kModePartition, 1>(a);
            if (pipe)
                return pk2 ? launch_general_pipe<32, 2, false, dmmdev::kModePartition, 2>(a)
                           : launch_general_pipe<32, 1, false, dmmdev::kModePartition, 2>(a);
            return pk2 ? launch_general<32, 2, false, dmmdev::kModePartition>(a) : launch_general<32, 1, false, dmmdev::kModePartition>(a);
        case dmmdev::kModeIntegerSort:
            if (pipe && pipe_mode == 1)
                return pk2 ? launch_general_pipe<32, 2, false, dmmdev::kModeIntegerSort, 1>(a)
                           : launch_general_pipe<32, 1, false, dmmdev::kModeIntegerSort, 1>(a);
            if (pipe)
                return pk2 ? launch_general_pipe<32, 2, false, dmmdev::kModeIntegerSort, 2>(a)
                           : launch_general_pipe<32, 1, false, dmmdev::kModeIntegerSort, 2>(a);
            return pk2 ? launch_general<32, 2, false, dmmdev::kModeIntegerSort>(a) : launch_general<32, 1, false, dmmdev::kModeIntegerSort>(a);
        default:
            return pk2 ? launch_general<32, 2, false, dmmdev::kModeSortAny>(a) : launch_general<32, 1, false, dmmdev::kModeSortAny>(a);
    }
}

}  // namespace dmmhost
