"""Result-buffer reuse of the host API (CPU only): an array handed back by a
run is reused only after the caller dropped every reference to it."""
import numpy as np

from paper_2405_14430_b200 import _out_buffer


class _Owner:
    pass


def test_out_buffer_reused_only_when_released():
    o, x = _Owner(), np.zeros((8, 4))
    a = _out_buffer(o, x)
    b = _out_buffer(o, x)
    assert a is not b
    ida = id(a)
    view = a[2:]
    del a
    c = _out_buffer(o, x)          # a's base is still referenced by `view`
    assert id(c) != ida and c is not b
    del view
    d = _out_buffer(o, x)          # now released
    assert id(d) == ida
    e = _out_buffer(o, np.zeros((2, 2)))  # other shapes never alias
    assert e.shape == (2, 2)
