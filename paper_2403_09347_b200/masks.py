"""Block-sparse grid masks (reference BlockGrid / BlockMask / mask_from_spec,
pkg/src/burstsim/masking.py:33-180).

A `GridMask` is a coarse n_query_blocks x n_key_blocks grid over the GLOBAL
score matrix with explicitly skipped cells; it composes with the causal flag of
the attention call.  Cells are equal (the reference's validate() requires the
block counts to divide the sequence, masking.py:135-139), so a score (query
position p, key position c) is hidden iff cell (p * nqb // N, c * nkb // N) is
skipped -- exactly BlockMask.allowed (masking.py:120-128).  The kernels receive
the grid as a device byte table plus cell extents in `burst_hop`.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import MaskError


@dataclass(frozen=True)
class GridMask:
    n_query_blocks: int
    n_key_blocks: int
    skip: frozenset = field(default_factory=frozenset)
    total: int = 0            # global sequence length the cells tile (set by `bind`)

    def __post_init__(self):
        # BlockGrid.__post_init__ (masking.py:41-46)
        if self.n_query_blocks < 1 or self.n_key_blocks < 1:
            raise MaskError("block grid needs at least one block per axis")
        for qb, kb in self.skip:
            if not (0 <= qb < self.n_query_blocks and 0 <= kb < self.n_key_blocks):
                raise MaskError(f"skip cell ({qb}, {kb}) outside grid")

    @staticmethod
    def from_spec(spec) -> tuple["GridMask | None", bool]:
        """mask_from_spec (masking.py:150-180): None / "none" / "causal" / dict /
        JSON file path.  Returns (grid or None, causal flag)."""
        if spec is None or spec == "none":
            return None, False
        if spec == "causal":
            return None, True
        if isinstance(spec, (str, Path)):
            path = Path(spec)
            if not path.exists():
                raise MaskError(f"mask {spec!r} is neither 'none', 'causal', nor an existing file")
            try:
                spec = json.loads(path.read_text())
            except json.JSONDecodeError as e:
                raise MaskError(f"mask file {path}: invalid JSON ({e})")
        if not isinstance(spec, dict):
            raise MaskError(f"unsupported mask spec {spec!r}")
        try:
            g = GridMask(int(spec["n_query_blocks"]), int(spec["n_key_blocks"]),
                         frozenset((int(q), int(k)) for q, k in spec.get("skip", [])))
        except KeyError as e:
            raise MaskError(f"mask spec missing key {e.args[0]!r}")
        return g, bool(spec.get("causal", False))

    def bind(self, total: int) -> "GridMask":
        """The grid over a global sequence of `total` positions (validate's
        divisibility rule, masking.py:135-139)."""
        if total >= 2 ** 31:
            raise MaskError("grid masks support global lengths below 2^31 positions")
        if total % self.n_query_blocks or total % self.n_key_blocks:
            raise MaskError(f"grid {self.n_query_blocks}x{self.n_key_blocks} does not divide "
                            f"score matrix {total}x{total}")
        return GridMask(self.n_query_blocks, self.n_key_blocks, self.skip, total)

    @property
    def qcell(self) -> int:
        return self.total // self.n_query_blocks

    @property
    def kcell(self) -> int:
        return self.total // self.n_key_blocks

    def table(self) -> np.ndarray:
        t = np.zeros((self.n_query_blocks, self.n_key_blocks), dtype=np.uint8)
        for qb, kb in self.skip:
            t[qb, kb] = 1
        return t

    def allowed(self, q_pos, k_pos) -> np.ndarray:
        """Element map for explicit global positions (masking.py:110-130)."""
        q_pos, k_pos = np.asarray(q_pos), np.asarray(k_pos)
        return self.table()[(q_pos // self.qcell)[:, None], (k_pos // self.kcell)[None, :]] == 0

    def validate(self, causal: bool, real_rows: int | None = None) -> None:
        """Reject masks that leave a real query row with no visible key
        (BlockMask.validate, masking.py:132-147)."""
        key = (causal, real_rows)
        done = _VALIDATED.setdefault(self, set())
        if key in done:
            return
        n = self.total
        rows = n if real_rows is None else real_rows
        t = self.table()
        kc = np.arange(rows) // self.kcell        # padded keys are masked off (with_padding)
        for qb in range(self.n_query_blocks):
            r0, r1 = qb * self.qcell, min((qb + 1) * self.qcell, rows)
            if r0 >= r1:
                continue
            open_cols = t[qb][kc] == 0             # visible key positions for this cell row
            if causal:
                # first visible key of each row r must be <= r
                first = int(np.argmax(open_cols)) if open_cols.any() else n
                if first > r0:
                    raise MaskError(f"query row {r0} has every key masked out")
            elif not open_cols.any():
                raise MaskError(f"query row {r0} has every key masked out")
        done.add(key)

    def device_table(self, device):
        """Cached uint8 [nqb * nkb] table on `device` (the burst_hop grid_skip)."""
        import torch
        key = (str(device),)
        cache = _TABLES.setdefault(self, {})
        if key not in cache:
            t = torch.from_numpy(self.table().reshape(-1).copy()).to(device)
            # the table is shared by every stream that launches with this mask (the rank
            # threads of run_ring_pass each run on their own stream): the H2D copy was
            # only ordered on the creating thread's stream, so finish it before any
            # other stream can see the cached tensor
            torch.cuda.current_stream(t.device).synchronize()
            cache[key] = t
        return cache[key]


_TABLES: dict = {}
_VALIDATED: dict = {}
