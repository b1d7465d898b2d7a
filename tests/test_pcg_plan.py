"""Host logic of the PCG plan's partition (csrc/pcg.cu PcgPlan::build): the
bisection with aggregate-aligned splits and the Lloyd relaxation of its
subdomains. CPU only: nrr_debug_pcg_partition makes no device call."""
import ctypes as C

import numpy as np
import pytest

from paper_2206_03410_b200 import capi
from paper_2206_03410_b200 import registration as R
from tests.helpers import strip_problem


def partition(p, sms):
    lib = capi.load()
    v = p.view()
    N = p.graph.node_count
    out3 = np.zeros(3, np.int32)
    row_begin = np.zeros(sms + 1, np.int32)
    row_node = np.zeros(N, np.int32)
    capi.check(lib.nrr_debug_pcg_partition(C.byref(v), sms, capi.i(out3), capi.i(row_begin), capi.i(row_node)))
    grid = int(out3[0])
    return grid, int(out3[1]), int(out3[2]), row_begin[:grid + 1].copy(), row_node


def halo_sizes(p, row_begin, row_node):
    N = p.graph.node_count
    label = np.empty(N, int)
    for g in range(len(row_begin) - 1):
        label[row_node[row_begin[g]:row_begin[g + 1]]] = g
    touched = [set() for _ in range(len(row_begin) - 1)]
    for a, b in p.graph.edges:
        if label[a] != label[b]:
            touched[label[a]].add(b)
            touched[label[b]].add(a)
    return np.array([len(t) for t in touched])


@pytest.fixture(scope="module")
def sheet():
    return strip_problem(90, 90, seed=5, mult=2.2)  # ~1.6K nodes


def test_partition_is_a_permutation_with_capped_subdomains(sheet):
    N = sheet.graph.node_count
    grid, agg, max_rows, rb, rn = partition(sheet, 148)
    assert grid == min(148, N)
    assert sorted(rn.tolist()) == list(range(N))
    sizes = np.diff(rb)
    assert rb[0] == 0 and rb[-1] == N and sizes.min() >= 1
    assert sizes.max() == max_rows
    mean = -(-N // grid)
    assert max_rows <= max(mean + -(-mean * 10 // 100), 24)  # 10% above the mean (or the bisection's own maximum)
    assert agg == 4


def test_partition_is_deterministic(sheet):
    a = partition(sheet, 148)
    b = partition(sheet, 148)
    assert a[:3] == b[:3] and np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])


def test_relaxation_shortens_the_interfaces(sheet, monkeypatch):
    _, _, _, rb1, rn1 = partition(sheet, 148)
    monkeypatch.setenv("NRR_LLOYD", "0")
    _, _, _, rb0, rn0 = partition(sheet, 148)
    h1, h0 = halo_sizes(sheet, rb1, rn1), halo_sizes(sheet, rb0, rn0)
    assert h1.sum() < 0.95 * h0.sum()  # rounder subdomains: fewer halo rows in total
    assert h1.max() <= h0.max()


def test_aggregates_are_subtrees_of_the_bisection(sheet, monkeypatch):
    """Without the relaxation the subdomains of one aggregate (4 consecutive
    CTAs) form a box of the aligned bisection: their joint bounding boxes
    overlap far less than those of unaligned groups of 4."""
    monkeypatch.setenv("NRR_LLOYD", "0")
    pos = sheet.graph.node_positions

    def overlap(align):
        monkeypatch.setenv("NRR_RCB_ALIGN", str(align))
        grid, agg, _, rb, rn = partition(sheet, 148)
        boxes = []
        for g0 in range(0, grid, agg):
            ids = rn[rb[g0]:rb[min(g0 + agg, grid)]]
            boxes.append((pos[ids].min(0), pos[ids].max(0)))
        tot = 0.0
        for i in range(len(boxes)):
            for j in range(i + 1, len(boxes)):
                lo = np.maximum(boxes[i][0], boxes[j][0])
                hi = np.minimum(boxes[i][1], boxes[j][1])
                ext = np.clip(hi - lo, 0, None)
                tot += ext[0] * ext[1]  # the sheet lies in x, y
        return tot

    assert overlap(4) < 0.5 * overlap(1) + 1e-12


def test_small_graphs(monkeypatch):
    p = strip_problem(8, 5, seed=1, mult=2.2)
    N = p.graph.node_count
    for sms in (1, 3, 148):
        grid, agg, max_rows, rb, rn = partition(p, sms)
        assert grid == min(sms, N)
        assert sorted(rn.tolist()) == list(range(N))
        assert np.diff(rb).min() >= 1
