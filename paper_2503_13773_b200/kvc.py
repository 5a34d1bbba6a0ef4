"""kvc.BlockPool (kvc.py:55-375) backed by the device pool.

Every mutation runs on the GPU through the engine's own pool functions
(csrc/pool_ops.cuh via csrc/pool_api.cuh, one single-thread kernel per
operation), including the N1 block tables under them; this class only maps
request ids to record slots, turns the device's contract codes into the
reference's ValueErrors, and packs Grant / Shortfall / EmbedQuote.  It is the
white-box surface the reference's own BlockPool tests drive
(tests/test_pool_device.py); the engine itself keeps its pool resident and
never goes through it."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Tuple, Union

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class Grant:
    tokens: int
    footprint: int


@dataclass(frozen=True)
class Shortfall:
    missing: int


AllocResult = Union[Grant, Shortfall]


@dataclass(frozen=True)
class EmbedQuote:
    host: int
    start_offset: int
    feasible_slack: int


OP_ALLOCATE, OP_EMBED, OP_DRAW_RESERVED, OP_GROW, OP_PROMOTE, OP_RELEASE, OP_SET_USED, OP_GAIN = range(8)


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


class BlockPool:
    """Token pool owned by the engine loop; all operations are sequential
    (kvc.py:55).  max_records bounds the distinct request ids it can hold."""

    def __init__(self, capacity: int, block_size: int = 8, reserved_blocks: int = 8, buffer_b: int = 8,
                 allow_stacking: bool = False, max_records: int = 4096, device: int = 0) -> None:
        lib = N.load()
        h = C.c_void_p()
        rc = lib.co_pool_create(int(capacity), int(block_size), int(reserved_blocks), int(buffer_b),
                                int(bool(allow_stacking)), int(max_records), int(device), C.byref(h))
        if rc == N.CO_EINVAL:
            raise ValueError(lib.co_last_error().decode())
        N.check(rc, "co_pool_create")
        self._lib = lib
        self._h = h
        self.capacity = capacity
        self.block_size = block_size
        self.reserved_target = reserved_blocks
        self.buffer_b = buffer_b
        self.allow_stacking = allow_stacking
        self._slot: Dict[int, int] = {}
        self._id: List[int] = []
        self._max = max_records
        self._out = np.zeros(4, dtype=np.int64)
        self._sc = np.zeros(6, dtype=np.int64)
        self._rec = np.zeros((max_records, 9), dtype=np.int64)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.co_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- slots ----------------------------------------------------------------

    def _slot_of(self, req_id: int, create: bool) -> int:
        s = self._slot.get(req_id)
        if s is None:
            if not create:
                return -1
            if len(self._id) >= self._max:
                raise ValueError(f"device pool holds at most {self._max} distinct request ids")
            s = self._slot[req_id] = len(self._id)
            self._id.append(req_id)
        return s

    def _op(self, op: int, req_id: int, a: int = 0, b: int = 0, c: int = 0, ids=()) -> Tuple[int, int, int]:
        s = self._slot_of(req_id, create=op in (OP_ALLOCATE, OP_EMBED, OP_DRAW_RESERVED))
        if s < 0:
            raise ValueError(f"no allocation for request {req_id}")
        N.check(self._lib.co_pool_op(self._h, op, s, int(a), int(b), int(c), _i64p(self._out)), "co_pool_op")
        code, x, y = (int(v) for v in self._out[:3])
        if code < 0:
            raise ValueError(self._message(-code, req_id, a, x, ids))
        return code, x, y

    @staticmethod
    def _message(pv: int, req_id: int, a: int, x: int, ids) -> str:
        host = ids[0] if ids else None
        return {
            1: "n_tokens must be >= 1",
            2: f"request {req_id} already holds an allocation",
            3: f"no allocation for request {req_id}",
            4: f"no allocation for request {host}",
            5: f"host {host} is itself embedded",
            6: "a request cannot host itself",
            7: f"host {host} already has a guest",
            8: "embed region exceeds host allocation",
            9: "embed region overlaps an existing guest",
            10: "n_blocks must be >= 1",
            11: "guests cannot draw from the reserve",
            12: f"request {req_id} is not embedded",
            13: f"request {req_id}: used {a} outside [0, {x}]",
        }.get(pv, f"device pool contract violation {pv}")

    def _state(self, records: bool = False) -> None:
        N.check(self._lib.co_pool_state(self._h, _i64p(self._sc), _i64p(self._rec) if records else None),
                "co_pool_state")

    def _record(self, req_id: int) -> np.ndarray:
        s = self._slot.get(req_id, -1)
        self._state(records=True)
        if s < 0 or not self._rec[s, 0]:
            raise ValueError(f"no allocation for request {req_id}")
        return self._rec[s]

    # -- derived state (kvc.py:88-152) ------------------------------------------

    @property
    def free_tokens(self) -> int:
        self._state()
        return int(self._sc[0])

    @property
    def footprint_tokens(self) -> int:
        self._state()
        return int(self._sc[1])

    @property
    def granted_tokens(self) -> int:
        self._state()
        return int(self._sc[2])

    @property
    def used_tokens(self) -> int:
        self._state()
        return int(self._sc[3])

    @property
    def reserved_blocks_current(self) -> int:
        self._state()
        return int(self._sc[4])

    def owners(self) -> List[int]:
        self._state(records=True)
        live = [s for s in range(len(self._id)) if self._rec[s, 0]]
        return [self._id[s] for s in sorted(live, key=lambda s: self._rec[s, 8])]

    def holds(self, req_id: int) -> bool:
        s = self._slot.get(req_id, -1)
        if s < 0:
            return False
        self._state(records=True)
        return bool(self._rec[s, 0])

    def granted_of(self, req_id: int) -> int:
        return int(self._record(req_id)[1])

    def used_of(self, req_id: int) -> int:
        return int(self._record(req_id)[7])

    def host_of(self, req_id: int) -> Optional[int]:
        h = int(self._record(req_id)[2])
        return None if h < 0 else self._id[h]

    def guests_of(self, req_id: int) -> List[int]:
        r = self._record(req_id)
        out, g = [], int(r[5])
        while g >= 0:
            out.append(self._id[g])
            g = int(self._rec[g, 6])
        return out

    def offset_of(self, req_id: int) -> int:
        return int(self._record(req_id)[3])

    def reserved_drawn_of(self, req_id: int) -> int:
        return int(self._record(req_id)[4])

    def net_release_gain(self, req_id: int) -> int:
        return self._op(OP_GAIN, req_id)[1]

    # -- operations (kvc.py:156-332) --------------------------------------------

    @staticmethod
    def _result(code: int, x: int, y: int) -> AllocResult:
        return Grant(tokens=x, footprint=y) if code > 0 else Shortfall(missing=x)

    def allocate(self, req_id: int, n_tokens: int) -> AllocResult:
        return self._result(*self._op(OP_ALLOCATE, req_id, n_tokens))

    def find_embedding_host(self, running: Iterable[Tuple[int, int, int]], cand_prompt: int, cand_out: int,
                            buffer_b: Optional[int] = None) -> Optional[EmbedQuote]:
        b = self.buffer_b if buffer_b is None else buffer_b
        if b < 0:
            raise ValueError("buffer_b must be >= 0")
        rows = [(self._slot.get(h, -1), h, a, u) for h, a, u in running]
        tri = np.array(rows, dtype=np.int64).reshape(-1, 4)
        N.check(self._lib.co_pool_find_host(self._h, len(rows), _i64p(tri) if len(rows) else None, int(cand_prompt),
                                            int(cand_out), int(b), _i64p(self._out)), "co_pool_find_host")
        found, slot, start, slack = (int(v) for v in self._out)
        if not found:
            return None
        return EmbedQuote(host=self._id[slot], start_offset=start, feasible_slack=slack)

    def embed(self, req_id: int, n_tokens: int, quote: EmbedQuote) -> AllocResult:
        hs = self._slot.get(quote.host, -1)
        return self._result(*self._op(OP_EMBED, req_id, n_tokens, hs, quote.start_offset, ids=(quote.host,)))

    def draw_reserved(self, req_id: int, n_blocks: int) -> AllocResult:
        return self._result(*self._op(OP_DRAW_RESERVED, req_id, n_blocks))

    def grow(self, req_id: int, n_tokens: int) -> AllocResult:
        if n_tokens < 1:
            raise ValueError("n_tokens must be >= 1")
        return self._result(*self._op(OP_GROW, req_id, n_tokens))

    def promote_guest(self, req_id: int) -> AllocResult:
        return self._result(*self._op(OP_PROMOTE, req_id))

    def release(self, req_id: int) -> int:
        return self._op(OP_RELEASE, req_id)[1]

    def set_used(self, req_id: int, used_tokens: int) -> None:
        self._op(OP_SET_USED, req_id, used_tokens)

    # -- invariants (kvc.py:336-375) ---------------------------------------------

    def check_invariants(self) -> None:
        rc = self._lib.co_pool_check(self._h)
        if rc == N.CO_EDEVICE:
            raise ValueError(self._lib.co_last_error().decode())
        N.check(rc, "co_pool_check")

    def block_tables(self) -> Tuple[Dict[int, List[int]], List[int]]:
        """N1: {req_id: pages} of standalone records and the free stack."""
        lens = np.zeros(self._max, dtype=np.int32)
        n_pages = self.capacity // self.block_size
        pages = np.zeros(max(1, n_pages), dtype=np.int32)
        free = np.zeros(max(1, n_pages), dtype=np.int32)
        nf = C.c_int32()
        i32 = C.POINTER(C.c_int32)
        N.check(self._lib.co_pool_read_tables(self._h, lens.ctypes.data_as(i32), pages.ctypes.data_as(i32),
                                              len(pages), free.ctypes.data_as(i32), C.byref(nf)),
                "co_pool_read_tables")
        out, w = {}, 0
        for s, ln in enumerate(lens.tolist()):
            if ln:
                out[self._id[s]] = pages[w:w + ln].tolist()
            w += ln
        return out, free[:nf.value].tolist()
