"""B200-native integer-sort engine (LSD radix sort and n-bucket sort of arXiv 1206.3511).

Drop-in for the reference's sort path (proj/core/include/intsort/sort.hpp): the
same entry points, backed by hand-written sm_100a kernels behind the C ABI in
include/isort.h.  See DESIGN.md and INTEGRATION.md.
"""
from ._lib import CudaError, InvalidArgument, IsortError, SequenceIoError  # noqa: F401
from .intsort import (  # noqa: F401
    RECORD_DTYPE,
    RadixPlan,
    bucket_index,
    bucket_index_batch,
    bucket_sort,
    build_radix_plan,
    counting_sort_by_digit,
    extract_digit,
    insertion_sort,
    keys_of,
    radix_sort_lsd,
    seq_of,
    tags_of,
)
from .sequence import SequenceHeader, read_sequence, write_sequence  # noqa: F401  (sequence_io.hpp mirror)

__all__ = [
    "CudaError", "InvalidArgument", "IsortError", "RECORD_DTYPE", "RadixPlan", "bucket_index",
    "bucket_index_batch", "bucket_sort", "build_radix_plan", "counting_sort_by_digit", "extract_digit",
    "insertion_sort", "keys_of", "radix_sort_lsd", "seq_of", "tags_of",
    "SequenceHeader", "SequenceIoError", "read_sequence", "write_sequence",
]
