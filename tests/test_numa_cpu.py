"""NUMA placement policy on CPU (reference pool =
std::vector, proj/core/src/buffer_pool.cpp:10). Each engine places its pinned
ring on the GPU's NUMA node with MPOL_PREFERRED before the first touch and
binds its threads to that node; this checks the placement primitive the pool
uses with move_pages(2). Hosts with one node skip the placement check (the
policy is a no-op there) but still exercise the query path."""
import ctypes
import mmap

import pytest


def _buffer(length):
    m = mmap.mmap(-1, length, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
    return m, addr


def test_page_query_reports_a_node_for_touched_pages(lz):
    m, addr = _buffer(16 * 4096)
    try:
        m[:] = b"\x01" * len(m)
        nodes = lz.numa_page_nodes(addr, len(m))
        assert len(nodes) == 16
        assert all(0 <= n < lz.numa_node_count() for n in nodes), nodes
    finally:
        del addr
        m.close()


@pytest.mark.skipif("__import__('paper_2406_10707_b200').numa_node_count() < 2",
                    reason="single-NUMA-node host: placement is a no-op")
def test_preferred_node_places_pages_before_first_touch(lz):
    last = lz.numa_node_count() - 1
    m, addr = _buffer(64 * 4096)
    try:
        lz.numa_prefer_range(addr, len(m), last)
        m[:] = b"\x02" * len(m)  # first touch after the policy
        nodes = lz.numa_page_nodes(addr, len(m))
        assert nodes.count(last) == len(nodes), nodes
    finally:
        del addr
        m.close()
