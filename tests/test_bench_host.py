"""CPU checks of bench.py's host logic (no GPU, no library call): the N > 1 line guard keeps the
contract's JSON line when a measurement added after it stalls, and stays silent otherwise."""
import io
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_line_guard_prints_the_line_when_the_extras_stall():
    out, exits = io.StringIO(), []
    line = {"metric": "m", "value": 1.0}
    g = bench.LineGuard(line, 0, 0.05, exit_fn=exits.append, out=out)
    line["late"] = {"partial": True}   # keys added before the limit are kept
    time.sleep(0.3)
    assert exits == [0]
    d = json.loads(out.getvalue())
    assert d["value"] == 1.0 and d["extras_timeout_s"] == 0.05 and d["late"] == {"partial": True}
    assert g.finish() is False   # the caller must not print a second line


def test_line_guard_other_ranks_exit_without_printing():
    out, exits = io.StringIO(), []
    bench.LineGuard({"value": 1.0}, 3, 0.05, exit_fn=exits.append, out=out)
    time.sleep(0.3)
    assert exits == [0] and out.getvalue() == ""


def test_line_guard_is_silent_when_the_extras_finish():
    out, exits = io.StringIO(), []
    g = bench.LineGuard({"value": 1.0}, 0, 0.2, exit_fn=exits.append, out=out)
    assert g.finish() is True
    time.sleep(0.4)
    assert exits == [] and out.getvalue() == ""
