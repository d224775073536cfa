"""Result buffers of the host API (CPU only): a run writes into a fresh array
unless the caller hands one in with `out=`; the library never reuses an
array it returned (refcount-based reuse was unsafe)."""
import numpy as np
import pytest

from paper_2405_14430_b200 import ValidationError, _out_buffer


def test_out_buffer_fresh_unless_given():
    x = np.zeros((8, 4))
    a = _out_buffer(x)
    b = _out_buffer(x)
    assert a is not b and a.shape == x.shape and a.dtype == np.float64
    mine = np.empty((8, 4))
    assert _out_buffer(x, mine) is mine


@pytest.mark.parametrize("bad", [np.empty((8, 4), np.float32), np.empty((4, 8)),
                                 np.empty((8, 8))[:, :4], "nope"])
def test_out_buffer_rejects_mismatched_arrays(bad):
    with pytest.raises(ValidationError):
        _out_buffer(np.zeros((8, 4)), bad)
