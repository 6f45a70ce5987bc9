"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module generates INPUTS only (graphs, feature tables, seed lists); it
holds none of the method's arithmetic.  See ``synth.py`` and DESIGN.md
("Input recipe").
"""
from .synth import (CONFIGS, Workload, make_workload, make_graph, make_seeds, make_features, feature_rows,
                    feature_rows_np, config_rows, make_packed_lists)

__all__ = ["CONFIGS", "Workload", "make_workload", "make_graph", "make_seeds", "make_features", "feature_rows",
           "feature_rows_np", "config_rows", "make_packed_lists"]
