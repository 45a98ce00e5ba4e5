"""Simulated 1D device grid (TEST INFRASTRUCTURE).

The pattern of SPEC.md:22-118 (module `simgrid`): P devices are plain Python
lists of numpy arrays; collectives execute synchronously in device order
0..P-1; every call appends {primitive, bytes, participants} to a
comm log with the ring payload convention of
SPEC.md:109 — (P-1)/P x the full tensor bytes for AllGather / ReduceScatter /
All-to-All, 2(P-1)/P x for AllReduce — at a configurable bytes-per-element
(SPEC.md:108).  A memory ledger tracks live bytes per device.

Pins (tests/test_oracle_grid.py): SPEC.md:54-56, 63-65, 70-72, 79-81, 88-90
worked examples; identities of SPEC.md:103 (AG o RS == AR; A2A involution)
checked on random tensors against direct index bookkeeping.
"""
from __future__ import annotations

import numpy as np


class Grid:
    def __init__(self, p: int, capacity_bytes: int = 1 << 62):
        if p < 1:
            raise ValueError("p must be >= 1 (SPEC.md:43)")
        self.p = p
        self.capacity = capacity_bytes
        self.comm_log: list[dict] = []
        self.alloc = [0] * p
        self.peak = [0] * p
        self._live: dict[int, tuple[int, int, str]] = {}
        self._next = 0

    # ---------------- comm log ----------------
    def _log(self, prim: str, full_bytes: float, factor: float):
        self.comm_log.append({"primitive": prim,
                              "bytes": int(round(full_bytes * factor)),
                              "participants": list(range(self.p))})

    def _frac(self):
        return (self.p - 1) / self.p

    # ---------------- collectives ----------------
    def all_gather(self, shards, axis=0, bpe=2):
        """Every device holds the concatenation along `axis` in device order."""
        assert len(shards) == self.p
        full = np.concatenate(shards, axis=axis)
        self._log("AllGather", full.size * bpe, self._frac())
        return [full.copy() for _ in range(self.p)]

    def reduce_scatter(self, tensors, axis=0, bpe=2):
        """Elementwise sum over devices (in order 0..P-1), device d gets slice d."""
        assert len(tensors) == self.p
        if tensors[0].shape[axis] % self.p:
            raise ValueError("reduce_scatter: dim not divisible by p (SPEC.md:61)")
        acc = tensors[0].copy()
        for t in tensors[1:]:
            acc = acc + t
        self._log("ReduceScatter", acc.size * bpe, self._frac())
        return [c.copy() for c in np.split(acc, self.p, axis=axis)]

    def all_reduce(self, tensors, bpe=4):
        assert len(tensors) == self.p
        acc = tensors[0].copy()
        for t in tensors[1:]:
            acc = acc + t
        self._log("AllReduce", acc.size * bpe, 2 * self._frac())
        return [acc.copy() for _ in range(self.p)]

    def all_to_all(self, tensors, split_axis, concat_axis, bpe=2):
        """Device d receives chunk d of every source's split_axis, concatenated
        along concat_axis in source order."""
        assert len(tensors) == self.p
        if tensors[0].shape[split_axis] % self.p:
            raise ValueError("all_to_all: split dim not divisible by p (SPEC.md:77)")
        chunks = [np.split(t, self.p, axis=split_axis) for t in tensors]
        out = [np.concatenate([chunks[src][dst] for src in range(self.p)], axis=concat_axis)
               for dst in range(self.p)]
        self._log("AllToAll", tensors[0].size * bpe, self._frac())
        return out

    def ring_pass(self, tensors, step=1, bpe=2):
        """Device d receives the tensor of device (d - step) mod p."""
        out = [tensors[(d - step) % self.p].copy() for d in range(self.p)]
        self._log("RingPass", tensors[0].size * bpe, 1.0 if self.p > 1 else 0.0)
        return out

    def permute(self, blocks, dest, bpe=2):
        """Point-to-point exchange (SendRecv): blocks[r] is the list of blocks device r
        holds, dest[r][i] the device block i goes to.  Returns, per device, the blocks it
        receives ordered by (source device, block index).  The log records the mean
        bytes a device sends off-device (blocks staying on their device are free)."""
        out = [[] for _ in range(self.p)]
        moved = 0
        for r in range(self.p):
            for i, blk in enumerate(blocks[r]):
                out[dest[r][i]].append(blk.copy())
                if dest[r][i] != r:
                    moved += blk.size * bpe
        self.comm_log.append({"primitive": "SendRecv", "bytes": int(round(moved / self.p)),
                              "participants": list(range(self.p))})
        return out

    # ---------------- memory ledger ----------------
    def track(self, dev: int, nbytes: int, tag: str = "") -> int:
        if self.alloc[dev] + nbytes < 0:
            raise ValueError("allocation underflow (SPEC.md:93)")
        self.alloc[dev] += nbytes
        self.peak[dev] = max(self.peak[dev], self.alloc[dev])
        hid = self._next
        self._next += 1
        self._live[hid] = (dev, nbytes, tag)
        return hid

    def release(self, hid: int):
        dev, nbytes, _ = self._live.pop(hid)
        self.alloc[dev] -= nbytes

    def live_bytes(self, dev: int, tag: str | None = None) -> int:
        return sum(nb for (d, nb, t) in self._live.values()
                   if d == dev and (tag is None or t == tag))

    def primitives(self):
        return [e["primitive"] for e in self.comm_log]
