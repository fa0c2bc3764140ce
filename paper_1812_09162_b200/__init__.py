"""qadc-b200: B200-native Quicker ADC scan path (arXiv 1812.09162) behind the reference's search interface.

Only what the hot path needs lives here: ``csrc/`` (CUDA kernels + the C ABI of include/qadc.h),
the ctypes loader, the host-side mirror of the reference interface (``index``), the packed-layout
helpers (``layout``), seeded synthetic inputs (``synth``) and the multi-GPU shard/merge glue (``dist``).
"""
from ._lib import QadcError, QadcSpec, build, lib  # noqa: F401
from .index import (FlatIndex, IvfIndex, MultiGpuFlatIndex, MultiGpuIvfIndex, SearchParams, SearchResult, allocate_dims, build_ivf_lists, encode,  # noqa: F401
                    ivf_assign_encode, merge_topk_device, open_index, packed_bytes, scan_list)
from .layout import pack_list, unpack_list  # noqa: F401
