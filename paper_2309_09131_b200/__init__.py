"""B200-native FLYCOO all-mode spMTTKRP with dynamic remapping.

Drop-in for the reference package's hot path (modecycle.engine:
mttkrp_mode / sweep_all_modes / remap_store, modecycle.layout:
build_sharded / select_params) with the compute on hand-written sm_100a
CUDA kernels (libflycoo.so, C ABI in include/flycoo.h).
"""

from .engine import (REMAP_STRATEGIES, BufferOrderError, RemapCursors, ShardOverflowError,
                     TrafficCounters, mttkrp_mode, remap_store, sweep_all_modes)
from .coo import CooTensor, Element, parse_frostt, read_frostt, synth_tensor, write_frostt
from .io import FrosttParseError, load_factor_set, save_factor_set
from .factors import DeviceFactorSet
from .layout import (CheckResult, DeviceShardedTensor, PartitionPlan, PlanReport,
                     build_device_sharded, build_sharded, device_has_duplicates, plan_from_counts,
                     record_bytes, validate_plan)
from .params import (InfeasibleParamsError, PartitionParams, default_element_bytes,
                     device_params, element_size_bits, select_params)
from .schedule import ScheduleMap, load_stats, schedule_super_shards
from .cpals import CpalsConfig, CpalsResult, cp_als, fit, normalize_factors

# reference-compatible names (FactorSet.random reproduces the reference's
# Philox stream; build_sharded takes the reference's (tensor, params))
FactorSet = DeviceFactorSet
ShardedTensor = DeviceShardedTensor

__version__ = "0.1.0"
