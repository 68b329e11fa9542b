"""paper_2411_06158_b200 -- B200-native batched IVF-MRQ search (arXiv 2411.06158).

Thin Python binding over the C ABI of libmrq (include/mrq.h): the functions
here only marshal arguments; every step of the query path runs in the CUDA
kernels of csrc/.  There is no CPU fallback: importing works everywhere, but
any call raises if libmrq.so is missing or no GPU is present.
"""
from .mrq import (  # noqa: F401
    MRQ_MODES, MRQError, SearchParams, Stats, lib, mrq_debug_fetch, mrq_debug_set, mrq_free, mrq_index_info, mrq_index_load,
    mrq_last_error, mrq_search_batch, mrq_search_batch_device, Index, mrq_nccl_unique_id, nccl_unique_id,
    mrq_shard_plan, mrq_build_gpu, BuildParams,
)
