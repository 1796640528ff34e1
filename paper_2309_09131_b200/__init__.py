"""B200-native FLYCOO all-mode spMTTKRP with dynamic remapping.

Drop-in for the reference package's hot path (modecycle.engine:
mttkrp_mode / sweep_all_modes / remap_store, modecycle.layout:
build_sharded / select_params) with the compute on hand-written sm_100a
CUDA kernels (libflycoo.so, C ABI in include/flycoo.h).
"""

from .engine import (REMAP_STRATEGIES, BufferOrderError, RemapCursors, ShardOverflowError,
                     TrafficCounters, mttkrp_mode, remap_store, sweep_all_modes)
from .factors import DeviceFactorSet
from .layout import (DeviceShardedTensor, PartitionPlan, build_device_sharded, plan_from_counts,
                     record_bytes)
from .params import (InfeasibleParamsError, PartitionParams, default_element_bytes,
                     device_params, element_size_bits, select_params)
from .schedule import ScheduleMap, load_stats, schedule_super_shards
from .cpals import CpalsConfig, CpalsResult, cp_als, fit, normalize_factors

# reference-compatible aliases
FactorSet = DeviceFactorSet
ShardedTensor = DeviceShardedTensor
build_sharded = build_device_sharded

__version__ = "0.1.0"
