"""Paged Stashing buffer (the reference's PagedStash,
pkg/src/moelab/planners.py:394-463) on the device.

Layers compute in ONE shared worst-case tmp buffer set; `stash` copies a layer's actual rows
(a device count, so no host sync) into fixed-size pages popped from the head of a circular
free list, `reload` copies them back and returns the pages to the tail. All of it is
stream-ordered kernels (csrc/stash.cu), so a multi-layer step can be captured in a CUDA
graph. Page accounting follows the reference exactly (tests/test_paged_stash.py replays the
reference's own op sequences against it).
"""
from __future__ import annotations

import torch

from . import _lib


def _stream():
    return torch.cuda.current_stream().cuda_stream


class PagedStashBuffer:
    """num_pages pages of page_rows rows; `widths` maps a saved tensor's name to its row
    width in bytes (one page pool per name, all indexed by the same page ids)."""

    def __init__(self, num_pages: int, widths: dict[str, int], page_rows: int = 64,
                 max_records: int = 64, max_pages_per_record: int | None = None,
                 worst_case_rows: int = 0, device=None):
        if num_pages < 1 or page_rows < 1:
            raise ValueError("num_pages and page_rows must be >= 1")
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.num_pages, self.page_rows = num_pages, page_rows
        self.worst_case_rows = worst_case_rows
        self.widths = dict(widths)
        for nm, w in self.widths.items():
            if w % 16:
                raise ValueError(f"row width of {nm!r} must be a multiple of 16 bytes")
        self.max_pages = max_pages_per_record or num_pages
        self.pools = {nm: torch.empty((num_pages * page_rows * w,), dtype=torch.uint8,
                                      device=dev) for nm, w in self.widths.items()}
        i32 = dict(dtype=torch.int32, device=dev)
        self.state = torch.empty((5,), **i32)
        self.ring = torch.empty((num_pages,), **i32)
        self.records = torch.zeros((max_records, 1 + self.max_pages), **i32)
        self._slot: dict[int, int] = {}  # live layer id -> record slot (host bookkeeping)
        self._free_slots = list(range(max_records))
        # overlap: stash copies on a "pack" stream while the next layer
        # computes, reloads prefetched on an "unpack" stream during the later layer's
        # backward; _dest keeps each record's reload destination + row count
        self.pack = torch.cuda.Stream(device=dev)
        self.unpack = torch.cuda.Stream(device=dev)
        self._dest: dict[int, tuple] = {}
        self._prefetched: dict[int, torch.cuda.Event] = {}
        self._stashed: dict[int, torch.cuda.Event] = {}  # pack-stream completion per record
        _lib.call("moe_stash_init", self.state.data_ptr(), self.ring.data_ptr(), num_pages,
                  _stream())

    def pages_needed(self, rows: int) -> int:
        return -(-rows // self.page_rows)

    def stash_async(self, layer_id: int, tensors: dict[str, torch.Tensor], rows_dev=None,
                    rows: int = 0) -> torch.cuda.Event:
        """stash() on the pack stream, ordered after the current stream's work so far.
        Returns the event after which the tensors may be overwritten (the caller must make
        the next writer of these buffers wait on it)."""
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        self.pack.wait_event(ev)
        with torch.cuda.stream(self.pack):
            self.stash(layer_id, tensors, rows_dev, rows)
            done = torch.cuda.Event()
            done.record(self.pack)
        self._stashed[layer_id] = done
        return done

    def prefetch(self, layer_id: int) -> bool:
        """Start the reload of a stashed record on the unpack stream, into the tensors it
        was stashed from (stash(..., keep_dest=True)), ordered after the current stream's
        work so far. reload() of that record then only waits for it."""
        if layer_id not in self._slot or layer_id not in self._dest or \
                layer_id in self._prefetched:
            return False
        tensors, rows_dev, rows = self._dest[layer_id]
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        self.unpack.wait_event(ev)
        st = self._stashed.pop(layer_id, None)
        if st is not None:  # the pages must have been written
            self.unpack.wait_event(st)
        with torch.cuda.stream(self.unpack):
            self._reload_now(layer_id, tensors, rows_dev, rows)
            done = torch.cuda.Event()
            done.record(self.unpack)
        self._prefetched[layer_id] = done
        return True

    def stash(self, layer_id: int, tensors: dict[str, torch.Tensor], rows_dev=None,
              rows: int = 0) -> torch.Tensor:
        """Copy rows [0, rows) of each named tensor into fresh pages. rows_dev: device int32
        scalar holding the row count (sync-free), else `rows`. Returns the device record
        [n_pages (-1: out of pages), page ids...]."""
        if layer_id in self._slot:
            raise ValueError(f"layer {layer_id} already stashed")
        if not self._free_slots:
            raise ValueError("too many live stash records")
        slot = self._free_slots.pop(0)
        self._slot[layer_id] = slot
        rec = self.records[slot]
        rd = rows_dev.data_ptr() if rows_dev is not None else None
        _lib.call("moe_stash_alloc", self.state.data_ptr(), self.ring.data_ptr(), self.num_pages,
                  self.page_rows, rd, int(rows), rec.data_ptr(), self.max_pages, _stream())
        for nm, t in tensors.items():
            self._copy(nm, t, rec, rd, rows, to_pages=True)
        self._dest[layer_id] = (dict(tensors), rows_dev, rows)
        return rec

    def reload(self, layer_id: int, tensors: dict[str, torch.Tensor], rows_dev=None,
               rows: int = 0) -> None:
        """Copy the layer's rows back into the given dense tensors, then free its pages (or,
        if prefetch() already did that into the same tensors, wait for it)."""
        ev = self._prefetched.pop(layer_id, None)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)
            return
        st = self._stashed.pop(layer_id, None)
        if st is not None:  # a stash_async record: its pages must have been written
            torch.cuda.current_stream().wait_event(st)
        self._reload_now(layer_id, tensors, rows_dev, rows)

    def _reload_now(self, layer_id, tensors, rows_dev, rows):
        slot = self._slot.pop(layer_id, None)
        if slot is None:
            raise KeyError(f"no stash record for layer {layer_id}")
        self._dest.pop(layer_id, None)
        rec = self.records[slot]
        rd = rows_dev.data_ptr() if rows_dev is not None else None
        for nm, t in tensors.items():
            self._copy(nm, t, rec, rd, rows, to_pages=False)
        _lib.call("moe_stash_release", self.state.data_ptr(), self.ring.data_ptr(),
                  self.num_pages, rec.data_ptr(), _stream())
        self._free_slots.append(slot)

    def release(self, layer_id: int) -> None:
        """Free a record's pages without copying (e.g. a failed or abandoned stash)."""
        slot = self._slot.pop(layer_id)
        self._dest.pop(layer_id, None)
        _lib.call("moe_stash_release", self.state.data_ptr(), self.ring.data_ptr(),
                  self.num_pages, self.records[slot].data_ptr(), _stream())
        self._free_slots.append(slot)

    def _copy(self, nm, t, rec, rd, rows, to_pages):
        w = self.widths[nm]
        if t.shape[-1] * t.element_size() != w or t.stride(-1) != 1:
            raise ValueError(f"{nm}: rows must be contiguous {w}-byte rows")
        max_rows = min(t.shape[0], self.max_pages * self.page_rows)
        _lib.call("moe_stash_copy", t.data_ptr(), t.stride(0) * t.element_size(),
                  self.pools[nm].data_ptr(), self.page_rows, w, rec.data_ptr(), rd, int(rows),
                  max_rows, int(to_pages), _stream())

    # ---- accounting (synchronising reads; planners.py:423-462 names) ----
    def stats(self) -> dict:
        head, free, peak, failed, last = self.state.tolist()
        return dict(head=head, free_pages=free, allocated_pages=self.num_pages - free,
                    peak_pages_used=peak, failed_stashes=failed, last_failed=bool(last))

    @property
    def free_pages(self) -> int:
        return self.stats()["free_pages"]

    @property
    def allocated_pages(self) -> int:
        return self.stats()["allocated_pages"]

    def peak_memory_rows(self) -> int:
        return self.worst_case_rows + self.stats()["peak_pages_used"] * self.page_rows

    def check(self) -> None:
        """Raise MemoryError (the reference's error) if any stash ran out of pages."""
        st = self.stats()
        if st["failed_stashes"]:
            raise MemoryError(f"out of pages: {st['failed_stashes']} stash(es) failed "
                              f"(free {st['free_pages']} of {self.num_pages})")
