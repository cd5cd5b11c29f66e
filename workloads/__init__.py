"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the CBC method (§III):
only tree topologies (parent arrays), seeded random tensors in the ABI leg
order, the BASELINE.json configs (B:7-11, readings in DESIGN.md) and the
circuit-layer operator construction of config 5 (A15).  Both `oracle/` and
`paper_2601_19650_b200/` import it; it imports neither.
"""
from .topology import (chain, complete_binary, star_of_chains_t3ns, star_of_chains_literal,
                       t_tree, ftps, children_of, depth_of, validate_parent)
from .generators import (random_tree_tensors, identity_operator, product_zero_state,
                         state_shapes, operator_shapes, complex_gaussian)
from .configs import CONFIGS, make_config, Instance
from .circuit import circuit_layer_operator, haar_unitary, layer_matching

__all__ = [
    "chain", "complete_binary", "star_of_chains_t3ns", "star_of_chains_literal", "t_tree", "ftps",
    "children_of", "depth_of", "validate_parent",
    "random_tree_tensors", "identity_operator", "product_zero_state", "state_shapes", "operator_shapes",
    "complex_gaussian", "CONFIGS", "make_config", "Instance",
    "circuit_layer_operator", "haar_unitary", "layer_matching",
]
