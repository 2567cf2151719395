"""paper_2010_12438_b200 — B200-native (sm_100a) policy-evaluation path of GO
(arXiv 2010.12438, "Transferable Graph Optimizers for ML Compilers").

A drop-in for the reference package's embed -> policy -> sample -> simulate path
(/root/reference/pkg/src/graphopt): same entry points and return types, computed by
hand-written CUDA kernels in libgo_b200.so (include/go_b200.h).  Nothing here falls
back to the CPU: without the library or a CUDA device the compute calls raise.
"""
from .config import (INVALID_REWARD, NUM_PRIORITY_LEVELS, TASK_ORDER, TASKS, EmbedConfig,
                     FusionConfig, PolicyConfig, PPOHyper, ordered_tasks)
from .costmodel import Topology, as_topology, kernel_time, uniform_topology
from .graph import OP_TYPES, Graph, GraphError, as_graph, feature_dim, node_features
from .params import ParamStore, init_all_params, randomize_zero_init

__all__ = [
    "EmbedConfig", "PolicyConfig", "FusionConfig", "PPOHyper", "TASK_ORDER", "TASKS",
    "NUM_PRIORITY_LEVELS", "INVALID_REWARD", "ordered_tasks", "Topology", "as_topology",
    "kernel_time", "uniform_topology", "OP_TYPES", "Graph", "GraphError", "as_graph",
    "feature_dim", "node_features", "ParamStore", "init_all_params", "randomize_zero_init",
]


def __getattr__(name):
    # heavy submodules (torch) are imported lazily
    import importlib
    for mod in ("embedding", "policy", "simulator", "training", "baselines"):
        m = importlib.import_module(f".{mod}", __name__)
        if hasattr(m, name):
            return getattr(m, name)
    raise AttributeError(name)
