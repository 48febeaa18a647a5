"""SceneFile JSON-lines: round trip, errors with line numbers."""
import numpy as np
import pytest

import paper_2511_17361_b200 as P
from paper_2511_17361_b200 import scenefile
from paper_2511_17361_b200.scenegen import gen_scene


def test_roundtrip_exact(tmp_path):
    b = gen_scene(5, 40, n_classes=4)
    classes = P.ClassTable(("a", "b", "c", "d"))
    p1, p2 = tmp_path / "s1.jsonl", tmp_path / "s2.jsonl"
    scenefile.write(str(p1), b, classes)
    scenefile.write(str(p2), b, classes)
    assert p1.read_bytes() == p2.read_bytes()
    r, cl = scenefile.read(str(p1))
    assert cl.names == classes.names
    for k in P.PrimitiveBatch.FIELDS:
        np.testing.assert_array_equal(getattr(r, k), getattr(b, k))   # bit-exact floats


def test_empty_and_errors(tmp_path):
    p = tmp_path / "e.jsonl"
    p.write_text('{"version": 1, "classes": ["x"]}\n')
    r, cl = scenefile.read(str(p))
    assert int(r.n_valid[0]) == 0
    p.write_text('{"version": 1, "classes": ["x"]}\n'
                 '{"mu": [0,0,0], "scale": [1,1,1], "quat": [1,0,0,0], "opacity": 1,'
                 ' "eps": [1,1], "logits": [NaN]}\n')
    with pytest.raises(ValueError, match=":2:"):
        scenefile.read(str(p))
    p.write_text('{"version": 1, "classes": ["x"]}\n{"mu": [0,0]}\n')
    with pytest.raises(ValueError, match=":2: malformed"):
        scenefile.read(str(p))
