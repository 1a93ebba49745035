"""Hierarchical rank layout (TEST INFRASTRUCTURE — see oracle/__init__.py).

P:69-70 (§3, Fig. 1): "The global network is divided into multiple groups, with
each group containing a single GPU from every node ... DASO creates groups
between GPUs with the same local identifier".  Node-local networks are "the
GPUs on each individual node".

Canonical dense rank map (reading R9 / SPEC S:38): rank = node * G + local.
"""
from __future__ import annotations


def check_cluster(num_nodes: int, gpus_per_node: int) -> None:
    if num_nodes < 1 or gpus_per_node < 1:
        raise ValueError("config error: num_nodes and gpus_per_node must be >= 1")


def rank_of(node: int, local: int, gpus_per_node: int) -> int:
    return node * gpus_per_node + local


def rank_lookup(rank: int, num_nodes: int, gpus_per_node: int) -> tuple[int, int]:
    """global rank -> (node, local).  Out-of-range rank -> range error."""
    check_cluster(num_nodes, gpus_per_node)
    if not 0 <= rank < num_nodes * gpus_per_node:
        raise IndexError("range error: rank out of [0, world)")
    return rank // gpus_per_node, rank % gpus_per_node


def node_groups(num_nodes: int, gpus_per_node: int) -> list[list[int]]:
    """node group j = the G ranks of node j."""
    check_cluster(num_nodes, gpus_per_node)
    return [[rank_of(j, l, gpus_per_node) for l in range(gpus_per_node)] for j in range(num_nodes)]


def global_groups(num_nodes: int, gpus_per_node: int) -> list[list[int]]:
    """group k = the GPU with local id k on every node, ascending node."""
    check_cluster(num_nodes, gpus_per_node)
    return [[rank_of(j, k, gpus_per_node) for j in range(num_nodes)] for k in range(gpus_per_node)]


def active_group(cycle_index: int, gpus_per_node: int) -> int:
    """P:79 "The role of global synchronization rotates between groups";
    order = ascending local id, round robin (reading R9)."""
    return cycle_index % gpus_per_node
