"""Canonical form of a skeleton result, shared by the golden-fixture maker (tools/make_golden.py) and
the GPU parity tests -- TEST INFRASTRUCTURE.

A result (skeleton + serial-rule sepsets + per-level counters + stop reason, skeleton.hpp:33-40) is
reduced to, per removal level l: the removed pairs (key = a * p + b, a < b, ascending) and their
sepset members (ascending vertex ids, core.hpp:302-306).  Level-0 pairs carry no members.  From that:
  * one SHA-256 per level over (keys, members), and one over the remaining edges;
  * a 64-bit hash per row a (sum over the row's removed pairs of a mixed (key, members) word, plus
    the row's adjacency bits), so a mismatch can be localised to rows without storing every pair.
Both the oracle's arrays (pyoracle.ResultArrays) and the device's SkeletonResult map to it.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def _mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser, elementwise on uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


@dataclass
class Canon:
    p: int
    edges: np.ndarray                       # int64 keys of the remaining edges, ascending
    blocks: dict = field(default_factory=dict)  # l -> (keys int64[n], members int32[n, l])
    counters: list = field(default_factory=list)  # (level, ci_tests, pseudo_inverses, edges_removed)
    stop_reason: str = ""

    def level_digest(self, ell: int) -> str:
        keys, mem = self.blocks.get(ell, (np.zeros(0, np.int64), np.zeros((0, ell), np.int32)))
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(keys, np.int64).tobytes())
        h.update(np.ascontiguousarray(mem, np.int32).tobytes())
        return h.hexdigest()

    def edges_digest(self) -> str:
        return hashlib.sha256(np.ascontiguousarray(self.edges, np.int64).tobytes()).hexdigest()

    def row_hash(self) -> np.ndarray:
        p = self.p
        out = np.zeros(p, np.uint64)
        with np.errstate(over="ignore"):
            for ell, (keys, mem) in self.blocks.items():
                if len(keys) == 0:
                    continue
                w = _mix(keys.astype(np.uint64) ^ (np.uint64(ell) << np.uint64(56)))
                for k in range(ell):
                    w = _mix(w ^ mem[:, k].astype(np.uint64))
                np.add.at(out, (keys // p).astype(np.int64), w)
            e = self.edges
            if len(e):
                np.add.at(out, (e // p).astype(np.int64), _mix(e.astype(np.uint64) + np.uint64(0x5555)))
        return out


def canon_from_oracle(r) -> Canon:
    """pyoracle.ResultArrays -> Canon."""
    p = r.p
    iu, ju = np.triu_indices(p, 1)
    keys_all = iu.astype(np.int64) * p + ju
    del iu, ju
    blocks = {}
    for ell in np.unique(r.slot_len[r.slot_len >= 0]):
        ell = int(ell)
        sel = np.nonzero(r.slot_len == ell)[0]
        keys = keys_all[sel]
        if ell:
            mem = r.members[r.slot_off[sel][:, None] + np.arange(ell)[None, :]].astype(np.int32)
        else:
            mem = np.zeros((len(sel), 0), np.int32)
        blocks[ell] = (keys, mem)
    edges = keys_all[r.slot_len < 0]
    counters = [(int(l.level), int(l.ci_tests), int(l.pseudo_inverses), int(l.edges_removed)) for l in r.levels]
    return Canon(p, edges, blocks, counters, r.stop_reason)


def canon_from_device(res) -> Canon:
    """paper_1812_08491_b200.SkeletonResult -> Canon (level-0 pairs = removed pairs not recorded at
    any level >= 1)."""
    p = res.skeleton.size()
    cells = res.skeleton.cells
    iu, ju = np.triu_indices(p, 1)
    keys_all = iu.astype(np.int64) * p + ju
    adj_up = cells[iu, ju].astype(bool)
    del iu, ju
    edges = keys_all[adj_up]
    removed = keys_all[~adj_up]
    blocks = {}
    recorded = []
    for ell, keys, mem in res.sepsets._blocks:
        blocks[int(ell)] = (np.asarray(keys, np.int64), np.asarray(mem, np.int32).reshape(len(keys), ell))
        recorded.append(np.asarray(keys, np.int64))
    lvl0 = np.setdiff1d(removed, np.concatenate(recorded)) if recorded else removed
    blocks[0] = (lvl0, np.zeros((len(lvl0), 0), np.int32))
    counters = [(int(l.level), int(l.ci_tests), int(l.pseudo_inverses), int(l.edges_removed)) for l in res.levels]
    return Canon(p, edges, blocks, counters, res.stop_reason.value)


def summary(c: Canon, full_levels=()) -> dict:
    """What a golden fixture stores (np.savez_compressed kwargs)."""
    out = {
        "p": np.int64(c.p),
        "counters": np.asarray(c.counters, np.uint64).reshape(-1, 4),
        "stop_reason": np.array(c.stop_reason),
        "edges_digest": np.array(c.edges_digest()),
        "edges_left": np.int64(len(c.edges)),
        "row_hash": c.row_hash(),
        "levels": np.asarray(sorted(c.blocks), np.int64),
        "level_digests": np.array([c.level_digest(l) for l in sorted(c.blocks)]),
    }
    for ell in full_levels:
        keys, mem = c.blocks.get(ell, (np.zeros(0, np.int64), np.zeros((0, ell), np.int32)))
        out[f"keys_{ell}"] = keys
        out[f"members_{ell}"] = mem.astype(np.uint16 if c.p < 65536 else np.int32)
    return out


def compare(dev: Canon, gold: dict) -> list[str]:
    """Differences between a device result and a stored fixture; [] when identical."""
    errs = []
    if dev.p != int(gold["p"]):
        return [f"p {dev.p} vs {int(gold['p'])}"]
    want = [tuple(int(v) for v in row) for row in gold["counters"]]
    if dev.counters != want:
        errs.append(f"counters {dev.counters} vs {want}")
    if dev.stop_reason != str(gold["stop_reason"]):
        errs.append(f"stop reason {dev.stop_reason} vs {gold['stop_reason']}")
    if len(dev.edges) != int(gold["edges_left"]) or dev.edges_digest() != str(gold["edges_digest"]):
        errs.append(f"remaining edges differ ({len(dev.edges)} vs {int(gold['edges_left'])})")
    for ell, dg in zip(gold["levels"], gold["level_digests"]):
        ell = int(ell)
        if dev.level_digest(ell) != str(dg):
            msg = f"level {ell} removals/sepsets differ"
            if f"keys_{ell}" in gold:
                gk, gm = gold[f"keys_{ell}"], gold[f"members_{ell}"].astype(np.int32)
                dk, dm = dev.blocks.get(ell, (np.zeros(0, np.int64), np.zeros((0, ell), np.int32)))
                common, gi, di = np.intersect1d(gk, dk, return_indices=True)
                diff_members = int((gm[gi] != dm[di]).any(axis=1).sum()) if ell else 0
                msg += (f": {len(gk) - len(common)} oracle-only pairs, {len(dk) - len(common)} device-only pairs, "
                        f"{diff_members} pairs with different sepsets")
            errs.append(msg)
    rh = dev.row_hash()
    bad = int((rh != gold["row_hash"]).sum())
    if bad:
        errs.append(f"{bad} of {dev.p} rows differ (row hash)")
    return errs
