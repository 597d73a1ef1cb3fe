"""hmx-b200: B200-native evaluation phase of MatRox (arXiv 1812.07152), Y = K~ W.

The hot path is ``hmx::evaluate`` (/root/reference/proj/src/executor.cpp:274-302),
rebuilt as sm_100a FP64 kernels behind the C-ABI in ``include/hmxg.h``.
"""
from .cds import CDS
from .executor import (Context, EvalPlan, EvalStats, Evaluator, HmxgError, PlanDefaults, evaluate,
                       generate_plan, plan_pseudocode)
from .instance import CONFIGS, Instance, InstanceSpec, build_instance, config

__all__ = [
    "CDS", "Context", "EvalPlan", "EvalStats", "Evaluator", "HmxgError", "PlanDefaults", "evaluate",
    "generate_plan", "plan_pseudocode", "CONFIGS", "Instance", "InstanceSpec", "build_instance", "config",
]
