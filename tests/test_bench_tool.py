"""CPU: tools/voxanim_bench.py -- the reference CLI's bench report format
(proj/src/cli.cpp:30-34 format_double = std::to_chars shortest, :299-312
bench_report_csv). The number cases were printed by std::to_chars (g++ 12,
libstdc++) for the listed doubles."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

from voxanim_bench import CSV_HEADER, bench_report_csv, format_double  # noqa: E402

TO_CHARS = [
    ("100", "100"),
    ("0.0001", "1e-04"),
    ("0.34179999999999999", "0.3418"),
    ("10000000000000000", "1e+16"),
    ("1234.5", "1234.5"),
    ("2.4999999999999999e-07", "2.5e-07"),
    ("123456789", "123456789"),
    ("0.5", "0.5"),
    ("1", "1"),
    ("10", "10"),
    ("0.001", "0.001"),
    ("0.01", "0.01"),
    ("12345678901234568", "12345678901234568"),
    ("1.0000000000000001e-05", "1e-05"),
    ("3e+21", "3e+21"),
    ("0.10000000000000001", "0.1"),
    ("1e+22", "1e+22"),
    ("1e+21", "1e+21"),
    ("-4206744482.576539", "-4206744482.576539"),
    ("28434449062617144", "28434449062617144"),
    ("0.00029283121089853807", "0.00029283121089853807"),
    ("-72.15303952570612", "-72.15303952570612"),
    ("0.009440659430614293", "0.009440659430614293"),
    ("34056376948438.574", "34056376948438.574"),
    ("1.1629223358228103e-07", "1.1629223358228103e-07"),
    ("-0", "-0"),
    ("5.3372049725616739e-09", "5.337204972561674e-09"),
    ("-1912550494540.0164", "-1912550494540.0164"),
    ("-86375838446.368378", "-86375838446.36838"),
    ("1424081658.7440104", "1424081658.7440104"),
    ("41617051819619.023", "41617051819619.02"),
    ("-9.0258788272715124e-15", "-9.025878827271512e-15"),
    ("-1.5984918279752366e-13", "-1.5984918279752366e-13"),
    ("51850494348766576", "51850494348766576"),
    ("17.056566199540327", "17.056566199540327"),
    ("7.5313060286093947", "7.531306028609395"),
    ("-3.6610513885406075e+18", "-3661051388540607488"),
    ("7.6877975345081477e-05", "7.687797534508148e-05"),
    ("54755289816349.305", "54755289816349.305"),
    ("3.4182311026980141e-06", "3.418231102698014e-06"),
    ("-553615.13563908311", "-553615.1356390831"),
    ("162.62541906132458", "162.62541906132458"),
    ("-12536448", "-12536448"),
    ("39694.009054883827", "39694.00905488383"),
    ("-76135655143691.078", "-76135655143691.08"),
    ("9.696685457359501e-06", "9.696685457359501e-06"),
    ("-1987466090630", "-1987466090630"),
    ("2.7943522155578547e-13", "2.7943522155578547e-13"),
]


def test_format_double_matches_to_chars():
    for text, expected in TO_CHARS:
        assert format_double(float(text)) == expected, text


def test_bench_report_csv_layout():
    out = bench_report_csv("animated-opt", [0.5, 0.25], {"rays": 10, "sphere_tests": 20, "svo_traversals": 3,
                                                         "pixels_reused": 4})
    assert out.splitlines() == [CSV_HEADER, "animated-opt,0,0.5,10,20,3,4", "animated-opt,1,0.25,10,20,3,4",
                                "animated-opt,0.375,2666.6666666666665"]


def test_acceptance_fixture_builds_and_loads(tmp_path):
    """tools/acceptance_perf.py's fixture: the reference acceptance models and
    scene documents, built with this library and read back by load_scene_file."""
    import paper_1911_06001_b200 as vx
    from acceptance_perf import build_fixture

    build_fixture(vx, str(tmp_path))
    bench = vx.Scene.load(str(tmp_path / "bench.json"), 640, 480)
    single = vx.Scene.load(str(tmp_path / "single.json"), 320, 240)
    assert bench.object_count() == 4 and single.object_count() == 1
    bench.evaluate(0.5)
    assert bench.get_object(2)[2] and not bench.get_object(0)[2]  # the tracked object moved, the static one not
