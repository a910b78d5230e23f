"""The Jacobi strip kernel's tile queue (csrc/jacobi.cu StripPlan), checked on
the host through sdfgb_debug_strip_tiles: for whole planes, multi-GPU slabs
and the edge / interior bands of the overlapped schedule, the persistent
warps' queue must cover every strip's output rows exactly once, in tiles
tall enough that a tile's unrolled prologue never meets plane row M-1."""
import ctypes

import numpy as np
import pytest

from paper_1902_10345_b200 import _lib

KSPX = 112  # kept columns per strip


@pytest.mark.parametrize("M,N,r0,r1,resident", [
    (8192, 8192, 0, 8192, 2368),     # J1, one wave of 148 x 16 warps
    (8192, 8192, 0, 8192, 64),       # few warps: tall tiles dominate
    (1000, 1000, 0, 1000, 2368),     # more warps than tall tiles: all short
    (1038, 8192, 7, 1031, 2368),     # a multi-GPU slab's owned rows
    (1038, 8192, 7, 23, 2368),       # its 16-row edge band
    (1038, 8192, 23, 1015, 2368),    # its interior band
    (300, 256, 100, 108, 2368),      # the smallest band (8 rows)
    (16, 132, 0, 16, 2368),          # the smallest plane
    (4099, 1028, 0, 4099, 1184),     # ragged rows and strips
])
def test_queue_covers_every_row_once(M, N, r0, r1, resident):
    L = _lib.load()
    cap = 1 << 16
    buf = np.zeros(3 * cap, np.int32)
    n = L.sdfgb_debug_strip_tiles(M, N, r0, r1, resident, ctypes.c_void_p(buf.ctypes.data), cap)
    assert 0 < n <= cap
    tiles = buf[:3 * n].reshape(-1, 3)
    nstrips = (N + KSPX - 1) // KSPX
    cover = np.zeros((nstrips, M), np.int32)
    for s, y0, ye in tiles:
        assert 0 <= s < nstrips and r0 <= y0 < ye <= r1
        cover[s, y0:ye] += 1
        # >= 16 rows (>= 8 in a band thinner than 32 rows): the prologue
        # (2F+1 rounded to 3) then never reaches row M-1
        assert ye - y0 >= (16 if r1 - r0 >= 32 else min(8, r1 - r0)), (s, y0, ye)
    assert (cover[:, r0:r1] == 1).all() and cover[:, :r0].sum() == 0 and cover[:, r1:].sum() == 0
    # the border-column strips' tiles are queued first in each group
    assert set(tiles[:2, 0]) == {0, nstrips - 1}
