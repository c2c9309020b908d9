"""Host logic of the multicolour order (tests/coloring.py): validity on the five configs' stencils."""
import numpy as np
import pytest

import synth
from coloring import greedy_colors, is_valid


@pytest.mark.parametrize("name,red,ncol", [("C1", None, 2), ("C2", 64, 2), ("C3", 64, None), ("C4", 8, 2)])
def test_greedy_colouring_of_config_stencils(name, red, ncol):
    cfg = synth.CONFIGS[name] if red is None else synth.CONFIGS[name].reduced(red)
    seq = synth.HostSequence(cfg)
    hm = seq.matrix(1, seq.initial())
    col = greedy_colors(hm.n, hm.row_ptr, hm.col_idx)
    assert is_valid(hm.n, hm.row_ptr, hm.col_idx, col)
    if ncol:
        assert col.max() + 1 == ncol
    assert col.max() + 1 <= 9


def test_invalid_colouring_detected():
    rp = np.array([0, 2, 4]); ci = np.array([0, 1, 0, 1])
    assert not is_valid(2, rp, ci, np.array([0, 0]))
    assert is_valid(2, rp, ci, np.array([0, 1]))
