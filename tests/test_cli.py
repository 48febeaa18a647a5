"""The sqocc CLI (SPEC.md:550-619 cli-io, the commands on the voxelization
path): CPU checks here, device runs under -m gpu."""
import json

import numpy as np
import pytest

from paper_2511_17361_b200 import cli, sqoc


def test_gen_scene_is_seeded_and_byte_identical(tmp_path, capsys):
    a, b, c = (str(tmp_path / n) for n in ("a.jsonl", "b.jsonl", "c.jsonl"))
    assert cli.main(["gen-scene", "--seed", "7", "--n", "40", "--out", a]) == 0
    assert cli.main(["gen-scene", "--seed", "7", "--n", "40", "--out", b]) == 0
    assert cli.main(["gen-scene", "--seed", "8", "--n", "40", "--out", c]) == 0
    assert open(a, "rb").read() == open(b, "rb").read() != open(c, "rb").read()
    assert len(open(a).read().splitlines()) == 41
    assert cli.main(["gen-scene", "--seed", "1", "--n", "0", "--out", c, "--format", "json"]) == 0
    assert json.loads(capsys.readouterr().out.splitlines()[-1])["n"] == 0
    assert len(open(c).read().splitlines()) == 1  # n = 0: header only


def test_validation_failures_exit_nonzero_and_write_nothing(tmp_path, capsys):
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"version": 1, "classes": ["a"]}\n{"mu": [0, 0]}\n')
    out = tmp_path / "g.sqoc"
    assert cli.main(["voxelize", "--scene", str(bad), "--out", str(out)]) == 2
    assert "bad.jsonl:2" in capsys.readouterr().err  # the malformed record's line
    assert not out.exists()
    assert cli.main(["gen-scene", "--seed", "1", "--n", "-1", "--out", str(out)]) == 2
    with pytest.raises(SystemExit):
        cli.main(["voxelize", "--scene", str(bad), "--out", str(out), "--grid-dims", "1,2"])


@pytest.mark.gpu
def test_voxelize_metrics_bench_on_device(tmp_path, capsys):
    import paper_2511_17361_b200 as P
    from paper_2511_17361_b200 import scenefile
    scene = str(tmp_path / "s.jsonl")
    # (a negative first coordinate needs the --flag=value form)
    flags = ["--grid-origin=-8,-8,-1", "--grid-dims", "40,36,16", "--resolution", "0.4"]
    assert cli.main(["gen-scene", "--seed", "3", "--n", "120", "--out", scene] + flags) == 0
    g1, g2 = str(tmp_path / "g1.sqoc"), str(tmp_path / "g2.sqoc")
    for g in (g1, g2):
        assert cli.main(["voxelize", "--scene", scene, "--out", g, "--vo", "--oracle",
                         "--format", "json"] + flags) == 0
    rep = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rep["pairs"] > 0 and rep["max_abs_dvo"] >= 0.0
    assert open(g1, "rb").read() == open(g2, "rb").read()  # deterministic
    # the file holds what the API computes
    batch, classes = scenefile.read(scene)
    spec = P.VoxelGridSpec((-8.0, -8.0, -1.0), (40, 36, 16), 0.4)
    r = P.Voxelizer(spec, P.VoxelizeConfig(), len(classes))(batch, dense=True)
    g = sqoc.read(g1)
    want = r.labels[0].cpu().numpy()
    np.testing.assert_array_equal(g.labels, np.where(want == r.free_code, 255, want))
    np.testing.assert_array_equal(g.v_o, r.v_o[0].cpu().numpy())
    # self-comparison -> all 1.0
    assert cli.main(["metrics", "--pred", g1, "--gt", g2, "--format", "json"]) == 0
    m = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert m["iou"] == 1.0 and m["miou"] == 1.0
    assert m["rayiou"] and all(v == 1.0 for v in m["rayiou"].values())
    # mismatched dims -> error
    g3 = str(tmp_path / "g3.sqoc")
    assert cli.main(["voxelize", "--scene", scene, "--out", g3, "--grid-origin=-8,-8,-1",
                     "--grid-dims", "40,36,8"]) == 0
    assert cli.main(["metrics", "--pred", g1, "--gt", g3]) == 2
    assert cli.main(["bench", "--scene", scene, "--repetitions", "3", "--format", "json"]
                    + flags) == 0
    b = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    # (tiny grid: the windows already cover most of it, so no real speed-up)
    assert b["speedup_vs_oracle"] > 0 and b["wall_ms"]["voxelize"]["p50"] > 0
