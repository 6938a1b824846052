"""paper_1507_01391_b200 -- B200-native (sm_100a) bank-conflict-free partition, sort and
permutation kernels (Afshani & Sitchinava, arXiv 1507.01391), drop-in for the reference's
DMM algorithms (/root/reference/proj/include/dmm).  The compute lives in libdmm_b200.so
(include/dmm_gpu.h); this package is its Python mirror.
"""
from .dmm import (  # noqa: F401
    FLAG_EXT_PARTIAL_GROUPS, FLAG_NO_ENFORCE_PRE, FLAG_NONSTRICT, KIND_PARTITION, KIND_PERMUTE, KIND_SORT_U32,
    ORDER_ALT, ORDER_ALT_DESC, ORDER_ASC, ORDER_DESC, CapacityExceeded, ConflictViolation, CudaError,
    DivisibilityViolation, Error, GeneralStats, InvalidInstance, KeyOutOfRange, NotBijective, NotSquare, OutOfBounds,
    OverlappingViews, PackingOverflow, PermuteReports, PostconditionFailed, ShapeViolation, UnsupportedShape,
    as_uint32, gen_instances, gen_keys, multisplit, multisplit_count, multisplit_scatter_to, integer_sort_general, lib, partition_general, partition_short_wide,
    partition_square, permute, permute_into, permute_steps, short_wide_probe, sort_rows, sort_short_wide, sort_square, sort_tall, sort_wide_any, supported,
    to_column_major, to_row_major, transpose_square, version)
from . import instance  # noqa: F401,E402  (instance.hpp mirror: text format, run_algorithm)
from .instance import (  # noqa: F401,E402
    Instance, RunOutcome, RunReport, TraceIncomplete, csv_header, csv_line, gen_instance, instance_from_text,
    instance_to_text, load_instance, run_algorithm, run_algorithms, save_instance, validate_instance)
from . import schedule  # noqa: F401,E402  (layout.hpp offline schedules)
from .schedule import (  # noqa: F401,E402
    DeviceSchedule, Move, Schedule, apply_schedule, offline_schedule, schedule_from_text, schedule_to_text)
from . import trace  # noqa: F401,E402  (reference trace files: text format + offline audit)
