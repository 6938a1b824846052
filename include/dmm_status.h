/* dmm_status.h -- status codes shared by the B200 C ABI (dmm_gpu.h) and the
 * CPU oracle (oracle/dmm_oracle.h).
 *
 * One code per exception class of the reference's error hierarchy
 * (/root/reference/proj/include/dmm/core.hpp:59-78), so a C++ shim can rethrow
 * the same type the reference would have thrown.
 */
#ifndef DMM_STATUS_H
#define DMM_STATUS_H

typedef enum dmm_status {
    DMM_OK = 0,
    DMM_SHAPE_VIOLATION = 1,        /* dmm::ShapeViolation        core.hpp:72 */
    DMM_INVALID_INSTANCE = 2,       /* dmm::InvalidInstance       core.hpp:74 */
    DMM_KEY_OUT_OF_RANGE = 3,       /* dmm::KeyOutOfRange         core.hpp:73 */
    DMM_DIVISIBILITY_VIOLATION = 4, /* dmm::DivisibilityViolation core.hpp:75 */
    DMM_POSTCONDITION_FAILED = 5,   /* dmm::PostconditionFailed   core.hpp:76 */
    DMM_PACKING_OVERFLOW = 6,       /* dmm::PackingOverflow       core.hpp:77 */
    DMM_CAPACITY_EXCEEDED = 7,      /* dmm::CapacityExceeded      core.hpp:68 */
    DMM_NOT_SQUARE = 8,             /* dmm::NotSquare             core.hpp:70 */
    DMM_OUT_OF_BOUNDS = 9,          /* dmm::OutOfBounds           core.hpp:66 */
    DMM_OVERLAPPING_VIEWS = 10,     /* dmm::OverlappingViews      core.hpp:65 */
    DMM_ERROR = 11,                 /* dmm::Error (generic)       core.hpp:59 */
    DMM_NOT_BIJECTIVE = 12,         /* dmm::NotBijective          core.hpp:71 */
    DMM_CONFLICT_VIOLATION = 13,    /* dmm::ConflictViolation     core.hpp:63 */
    /* B200-side conditions with no reference counterpart */
    DMM_UNSUPPORTED_SHAPE = 64,     /* shape the reference accepts but no kernel is built for */
    DMM_INVALID_ARGUMENT = 65,      /* null pointer / zero count / bad flag */
    DMM_CUDA_ERROR = 66             /* launch or runtime failure (see dmm_last_error()) */
} dmm_status;

#endif /* DMM_STATUS_H */
