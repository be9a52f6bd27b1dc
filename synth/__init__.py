"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds ONLY input generation: graphs, features, labels, train masks,
partitions and initial weights.  It contains none of DIGEST's arithmetic (no
propagation values, no partition construction, no layer math), so it can serve
both sides of the parity tests without coupling them.
"""
from .configs import CONFIGS, GraphConfig, get_config, small_config
from .graphs import (make_graph, make_features, make_labels, make_train_mask,
                     make_weights, make_block_parts, make_random_parts, make_inputs,
                     SyntheticInputs)

__all__ = ["CONFIGS", "GraphConfig", "get_config", "small_config", "make_graph",
           "make_features", "make_labels", "make_train_mask", "make_weights",
           "make_block_parts", "make_random_parts", "make_inputs", "SyntheticInputs"]
