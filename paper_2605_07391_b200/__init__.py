"""B200-native MERBIT (arXiv 2605.07391): TILE preprocessing, descriptor-driven
SpMV and fused PageRank on sm_100a, behind the reference's merbit API.

The compute lives in libmerbit_b200.so (CUDA, C ABI: include/merbit_b200.h).
This package is the Python view of that ABI (tests, bench, multi-GPU
plumbing); C++ callers use include/merbit_b200/merbit.hpp.
"""
from .merbit import (BackendKind, BicgstabConfig, BicgstabResult, CapacityError, ConfigError, Context, CorruptionError,
                     CudaError, DeviceMatrix, DimensionError, DualBuffer, MerbitB200Backend,
                     MerbitError, PageRankConfig, PageRankPlan, PageRankResult, SimtConfig,
                     SpmvBackend, SpmvTrace, Tile, UnsupportedError, default_context,
                     device_count, generate_tile, generate_tile_for, make_backend,
                     merge_search, metadata_footprint, pagerank, plan_row_shards, recut_row_shards,
                     select_sigma, spmv_device, spmv_merbit, tile_counts, trace_counts,
                     bicgstab, solve_status_name)

__all__ = [
    "BackendKind", "BicgstabConfig", "BicgstabResult", "bicgstab", "solve_status_name",
    "CapacityError", "ConfigError", "Context", "CorruptionError", "CudaError",
    "DeviceMatrix", "DimensionError", "DualBuffer", "MerbitB200Backend", "MerbitError",
    "PageRankConfig", "PageRankPlan", "PageRankResult", "SimtConfig", "SpmvBackend",
    "SpmvTrace", "Tile", "UnsupportedError", "default_context", "device_count",
    "generate_tile", "generate_tile_for", "make_backend", "merge_search",
    "metadata_footprint", "pagerank", "plan_row_shards", "recut_row_shards", "select_sigma",
    "spmv_device",
    "spmv_merbit", "tile_counts", "trace_counts",
]
