"""The oracle pinned against the reference's own test suites.

oracle/port_tests/ ports proj/tests/test_{spatial,model,urdf,kinematics,
dynamics}.cpp (same seeds and tolerances: closed forms, known answers and
properties) plus the SPEC.md examples for control/batch onto the Eigen-free
restatement.  Each ported TEST_CASE is one pytest case here."""
import os
import subprocess

import pytest

import oracle_ffi


def _run():
    oracle_ffi.build()
    out = subprocess.run([oracle_ffi.PORT_TESTS], capture_output=True, text=True)
    results = {}
    detail = {}
    cur = []
    for line in out.stdout.splitlines():
        if line.startswith("RESULT "):
            body = line[len("RESULT "):]
            name, verdict = body.rsplit(" ", 1)
            results[name] = verdict
            detail[name] = "\n".join(cur)
            cur = []
        elif line.startswith("    "):
            cur.append(line)
    return results, detail


_RESULTS = None


def results():
    global _RESULTS
    if _RESULTS is None:
        _RESULTS = _run()
    return _RESULTS


def _case_names():
    src = os.path.join(oracle_ffi.ORACLE_DIR, "port_tests")
    names = []
    for f in sorted(os.listdir(src)):
        if not f.endswith(".cpp"):
            continue
        for line in open(os.path.join(src, f)):
            if line.startswith('TEST("'):
                suite, rest = line[len('TEST("'):].split('", "', 1)
                names.append(suite + "/" + rest.split('")', 1)[0])
    return names


@pytest.mark.parametrize("case", _case_names())
def test_reference_case(case):
    res, detail = results()
    assert case in res, f"{case} did not run"
    assert res[case] == "PASS", detail.get(case, "")


def test_all_cases_accounted():
    res, _ = results()
    assert len(res) >= 55
    assert all(v == "PASS" for v in res.values())
