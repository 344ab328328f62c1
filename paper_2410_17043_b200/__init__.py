"""B200-native Aurora MoE-layer hot path (arXiv 2410.17043), a drop-in behind
the reference package's scheduling / deployment API (``moeplan``).

Public surface mirrors the reference names used on the hot path:

* schedule (K2, on the GPU): ``build_schedule``, ``CommSchedule``, ``Phase``,
  ``DecompositionError``, ``validate_schedule``, ``bmax_*`` -- commsched.py
* domain types: ``TrafficMatrix``, ``ClusterSpec``, ``GpuSpec``, ``LayerProfile``,
  ``DeploymentPlan``, ``LoadVector``, ``deploy_to_gpus``, ``combine_colocated`` -- core.py
* deployment (host, once per model): ``assign_exclusive_hetero``,
  ``colocate_homogeneous``, ``colocate_heterogeneous``, ... -- placement.py
* the MoE layer engine itself (router, pack, schedule, NVSwitch
  dispatch/combine, tcgen05 experts, aggregation): ``AuroraMoELayer``
"""
from .commsched import (TIME_ATOL, CommSchedule, DecompositionError, Phase, ScheduleFn, ScheduleReport,
                        bmax_heterogeneous, bmax_homogeneous, build_schedule, decompose_raw,
                        validate_schedule)
from .core import (ClusterSpec, DeploymentPlan, GpuSpec, LayerProfile, LoadVector, TrafficMatrix,
                   combine_colocated, deploy_to_gpus, reverse_all_to_all, row_col_sums)
from .matching import Matching, bottleneck_matching, hopcroft_karp
from .placement import (CaseOnePreconditionError, assign_exclusive_hetero, colocate_heterogeneous,
                        colocate_homogeneous, colocated_pair_cost, expert_loads, pair_case1)

schedule_fn: ScheduleFn = build_schedule

__version__ = "0.1.0"


def __getattr__(name):  # the layer pulls in torch; import it lazily
    if name in ("AuroraMoELayer", "MoEConfig"):
        from . import layer
        return getattr(layer, name)
    raise AttributeError(name)
