"""Host logic of the dense tiling plan (csrc/dense_plan.h, pure integer C++): compiled into a
tiny host program with g++ and checked against its stated rules -- kernel kind by size,
configuration choice and fallback, look-ahead from the live-scratch budget, scratch ring
geometry.  No GPU needed."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include <cstdio>
#include "dense_plan.h"
using namespace ptdr;
int main() {
  const int nvs[] = {4, 5, 6, 8, 10, 11, 12, 13, 14, 15, 16};
  for (int nv : nvs) {
    const unsigned long long N = 1ull << nv;
    const unsigned long long xs[] = {N, N / 2, N / 8, 16, 32};
    for (unsigned long long x : xs) {
      for (int cfg = 0; cfg <= 8; ++cfg) {
        if (x == 0) continue;
        DensePlan p = make_dense_plan(nv, x, cfg, kSingleMax);
        printf("{\"nv\":%d,\"x\":%llu,\"req\":%d,\"kind\":%d,\"cfg\":%d,\"R\":%d,\"M\":%d,\"L\":%d,"
               "\"nslot\":%d,\"W\":%d,\"nchunks\":%llu,\"slot\":%llu,\"scratch\":%zu}\n",
               nv, x, cfg, p.kind, p.pipe_cfg, p.R, p.M, p.L, p.nslot, p.W,
               (unsigned long long)p.nchunks, (unsigned long long)p.slot_elems, p.scratch_bytes);
      }
    }
  }
  return 0;
}
'''


@pytest.fixture(scope="module")
def plans(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("plan")
    src = d / "plan.cpp"
    src.write_text(SRC)
    exe = d / "plan"
    subprocess.check_call([gxx, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "paper_2403_11644_b200", "csrc"),
                           str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True)
    return [json.loads(l) for l in out.splitlines()]


def test_kind_by_size(plans):
    for p in plans:
        if p["nv"] <= 5:
            assert p["kind"] == 0
        elif p["nv"] <= 10 and p["x"] % (4096 >> p["nv"]) == 0 and p["x"] >= 16:
            assert p["kind"] == 1, p
        elif p["nv"] >= 11:
            assert p["kind"] == 2, p


def test_default_configuration_and_fallback(plans):
    full = [p for p in plans if p["req"] == 1 and p["x"] == 1 << p["nv"] and p["kind"] == 2]
    assert full
    for p in full:
        if p["nv"] == 11:
            assert p["cfg"] == 4 and p["W"] == 32, p   # configuration 1 needs nv >= 12 (M >= 4)
        else:
            assert p["cfg"] == 1 and p["W"] == 16, p


def test_pipeline_geometry(plans):
    pipe = [p for p in plans if p["kind"] == 2 and p["cfg"] != 0]
    assert pipe
    for p in pipe:
        assert p["R"] + p["M"] == p["nv"] and 4 <= p["M"] <= 8, p
        assert p["x"] % p["W"] == 0 and p["nchunks"] == p["x"] // p["W"], p
        assert p["slot"] == p["W"] << p["nv"], p
        slot_bytes = p["slot"] * 16
        assert p["L"] == max(2, min(64, (40 << 20) // slot_bytes)), p
        ns = p["nslot"]
        assert ns & (ns - 1) == 0 and ns >= 1, p
        assert p["scratch"] == ns * slot_bytes, p
        # enough slots for the look-ahead unless the ring holds every chunk already
        assert ns >= min(p["L"] + 2, p["nchunks"]) or ns >= p["nchunks"], p
