"""Folding output (``sp_blocks``) -> the reference's Subgraph list.

``Subgraph`` semantics follow pruning.py:33-55: template_prefix, template
(member scopes of the lexicographically smallest instance in topological
order) and instances (prefix, member scopes) sorted by prefix.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class BlockArrays:
    """Host copy of a folding result, in the reference's block order."""

    block_T: np.ndarray
    block_inst_off: np.ndarray
    block_member_off: np.ndarray
    inst_prefix_node: np.ndarray
    inst_prefix_len: np.ndarray
    members: np.ndarray

    @classmethod
    def from_dict(cls, d: dict) -> "BlockArrays":
        return cls(**{k: d[k] for k in cls.__dataclass_fields__})

    @property
    def n_blocks(self) -> int:
        return len(self.block_T)

    def template_nodes(self, b: int) -> np.ndarray:
        o = int(self.block_member_off[b])
        return self.members[o: o + int(self.block_T[b])]

    def templates_csr(self):
        """(offsets, nodes) of every block's template (instance 0 rows)."""
        T = np.asarray(self.block_T, np.int64)
        off = np.zeros(len(T) + 1, np.int64)
        np.cumsum(T, out=off[1:])
        # block b's template = the first T[b] members from block_member_off[b]
        mo = np.asarray(self.block_member_off, np.int64)[:len(T)]
        src = np.repeat(mo - off[:-1], T) + np.arange(int(off[-1]), dtype=np.int64)
        nodes = np.asarray(self.members)[src].astype(np.int32, copy=False)
        return off, nodes

    def multiplicity(self, b: int) -> int:
        return int(self.block_inst_off[b + 1] - self.block_inst_off[b])


def prefix_of(low, node: int, length: int) -> str:
    o = int(low.name_off[node])
    return bytes(low.name_bytes[o: o + int(length)]).decode("utf-8")


def to_prune_doc(low, ba: BlockArrays) -> list:
    """[[template_prefix, template, [[prefix, members], ...]], ...] -- the same
    document tests/golden/make_golden.py records from the reference."""
    names = low.names
    out = []
    for b in range(ba.n_blocks):
        T = int(ba.block_T[b])
        i0, i1 = int(ba.block_inst_off[b]), int(ba.block_inst_off[b + 1])
        mo = int(ba.block_member_off[b])
        insts = []
        for r, j in enumerate(range(i0, i1)):
            pre = prefix_of(low, int(ba.inst_prefix_node[j]), int(ba.inst_prefix_len[j]))
            mem = [names[int(x)] for x in ba.members[mo + r * T: mo + (r + 1) * T]]
            insts.append([pre, mem])
        out.append([insts[0][0], list(insts[0][1]), insts])
    return out
