"""The reference's OWN test programs, linked against libtagc_b200 through the
reference-side adapter integration/hook_b200.cpp (a drop-in replacement for
proj/src/hook.cpp; recipe integration/Makefile, built by __graft_entry__.build
where /root/reference is present, the binaries travel with the repo):

* test_hook_b200: proj/tests/test_hook.cpp:55-361 unmodified — bit-exact
  integer round trip, 1-bit carry loss, ledger == model, bypass == baseline,
  theta 100, raw path, make_shards, validation errors — every exchange on the
  B200.
* acceptance_b200: proj/tests/acceptance.cpp criteria 1 (9 operating points x
  500 trials, W in {2,4,8}, acceptance.cpp:68-97), 2 (ledger == model on a
  real exchange, :101-150) and 7 (1-bit instability, :383-424), each
  tagc_reduce_shard call on the B200.

The host-only cases (policy shares, volume model, make_shards, validation)
also run in the CPU suite: no device is touched by them."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
HOOK = os.path.join(BUILD, "test_hook_b200")
ACC = os.path.join(BUILD, "acceptance_b200")

HOST_ONLY = ["gpt2-small parameter shares against the closed-form oracle",
             "policy none flags nothing, attention stays uncompressed",
             "volume model headline points", "exact volume model with explicit length",
             "make_shards partitions layers with round-robin owners",
             "geometry and validation failures propagate"]


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.relpath(path, ROOT)} not built (needs /root/reference at build time)")


def _run(args, timeout):
    r = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def test_reference_hook_tests_host_cases():
    _need(HOOK)
    for case in HOST_ONLY:
        rc, out = _run([HOOK, f"-tc={case}"], 120)
        assert rc == 0 and "1 passed" in out, out


@pytest.mark.gpu
def test_reference_hook_tests_on_b200():
    _need(HOOK)
    rc, out = _run([HOOK], 600)
    print(out)
    assert rc == 0, out
    assert "test cases: 15 | 15 passed | 0 failed" in out, out


@pytest.mark.gpu
@pytest.mark.parametrize("criterion", [1, 2, 7])
def test_reference_acceptance_on_b200(criterion):
    _need(ACC)
    rc, out = _run([ACC, "--only", str(criterion)], 1500)
    print(out)
    assert rc == 0, out
    assert f"[PASS] criterion {criterion}" in out and "[FAIL]" not in out, out
