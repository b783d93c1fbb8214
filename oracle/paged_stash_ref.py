"""Paged Stashing page allocator — CPU oracle, TEST INFRASTRUCTURE ONLY.

Restates the reference's PagedStash (pkg/src/moelab/planners.py:394-463):
  * fixed-size pages (page_size tokens), free list as a circular buffer (:402-406);
  * stash(layer, actual_tokens): ceil_div(actual, page_size) pages popped from the HEAD of
    the free list, recorded for the layer; MemoryError "out of pages" when short
    (:435-449); the high-water mark of allocated pages is tracked (:449);
  * reload(layer): the recorded pages are appended to the TAIL, in record order
    (:451-458);
  * peak_memory_tokens = worst_case_tokens + peak_pages_used * page_size (:460-462).
Pinned by tests/test_paged_stash.py against op sequences replayed through the reference
itself (tests/golden/make_stash_golden.py -> stash_golden.npz) and the reference's tests
(test_planners.py:314-375, test_acceptance.py:431-451).
"""
from __future__ import annotations


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


class PagedStashRef:
    def __init__(self, num_pages: int, page_size: int = 64, worst_case_tokens: int = 0):
        if num_pages < 1 or page_size < 1:
            raise ValueError("num_pages and page_size must be >= 1")
        self.num_pages = num_pages
        self.page_size = page_size
        self.worst_case_tokens = worst_case_tokens
        self.free = list(range(num_pages))
        self.records: dict[int, list[int]] = {}
        self.peak_pages_used = 0

    @property
    def free_pages(self) -> int:
        return len(self.free)

    @property
    def allocated_pages(self) -> int:
        return self.num_pages - len(self.free)

    def pages_needed(self, tokens: int) -> int:
        return ceil_div(tokens, self.page_size)

    def stash(self, layer: int, tokens: int) -> list[int]:
        if layer in self.records:
            raise ValueError(f"layer {layer} already stashed")
        need = self.pages_needed(tokens)
        if need > len(self.free):
            raise MemoryError(f"out of pages: need {need}, free {len(self.free)}")
        pages, self.free = self.free[:need], self.free[need:]
        self.records[layer] = pages
        self.peak_pages_used = max(self.peak_pages_used, self.allocated_pages)
        return list(pages)

    def reload(self, layer: int) -> list[int]:
        pages = self.records.pop(layer, None)
        if pages is None:
            raise KeyError(f"no stash record for layer {layer}")
        self.free.extend(pages)
        return pages

    def peak_memory_tokens(self) -> int:
        return self.worst_case_tokens + self.peak_pages_used * self.page_size
