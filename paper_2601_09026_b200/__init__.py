"""B200-native layer-parallel (MGRIT) training hot path of arxiv 2601.09026.

Drop-in for the reference mglp library's LayerStack / LayerParallelEngine /
controller API (see engine.py, controller.py); all compute runs in the
in-tree CUDA library _lib/libmglp_cuda.so (sm_100a, tcgen05 tensor cores).
"""
from ._native import ContractViolation, ValidationError  # noqa: F401
from .engine import (BackwardOutcome, ForwardOutcome, LayerParallelEngine,  # noqa: F401
                     LayerStack, PhaseTrace, SolveConfig, StackConfig, State, serial_adjoint,
                     serial_forward)
from .controller import (DeviceMonitor, IndicatorConfig, InexactnessMonitor,  # noqa: F401
                         ProbeScope, decide, last_pair_factor)

__all__ = ["StackConfig", "SolveConfig", "State", "LayerStack", "LayerParallelEngine",
           "serial_forward", "serial_adjoint", "PhaseTrace", "ForwardOutcome", "BackwardOutcome",
           "IndicatorConfig", "InexactnessMonitor", "DeviceMonitor", "ProbeScope", "decide",
           "last_pair_factor", "ValidationError", "ContractViolation"]
