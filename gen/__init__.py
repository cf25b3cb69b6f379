"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no shortest paths, no route
costs, no clustering): only graph topology/weights, SKU placement and order
lines, drawn from fixed seeds. See DESIGN.md "Input recipe".
"""
from .warehouse import (  # noqa: F401
    Graph, Orders, aisle, lattice, place_skus, zipf_orders, config, CONFIGS,
)
