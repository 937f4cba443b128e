"""B200-native executor of the AEGIS (arXiv 2604.03425) CKKS hot path.

The product is libaegis.so (hand-written sm_100a CUDA behind the C-ABI in
include/aegis.h); this package is its thin Python host binding.
"""
from .api import (BERT_PARAMS, SEED_INPUT, SEED_KEY, SEED_WEIGHT, AegisError, Bundle, Context,
                  Graph, LogicError, P2pWindow, Plan, graph_from_ops, plan_graph)

__all__ = ["BERT_PARAMS", "SEED_INPUT", "SEED_KEY", "SEED_WEIGHT", "AegisError", "Bundle",
           "Context", "Graph", "LogicError", "P2pWindow", "Plan", "graph_from_ops", "plan_graph"]
