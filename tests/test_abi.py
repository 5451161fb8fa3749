"""CPU checks of the C-ABI boundary (no compute calls on a device).

* libgsi_b200.so loads and exports every function include/gsi.h declares;
* the ctypes struct layouts equal the C layouts (sizeof/offsetof from a compiled probe);
* without a GPU every compute entry point fails loudly with GSI_ERR_CUDA (no CPU fallback);
* the host-side query-signature encoder agrees with the oracle's independent encoder.
"""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle
import workloads as W
from paper_1906_03420_b200 import gsi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_header_symbol():
    syms = gsi.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(gsi.lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", gsi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing


def _c_layout():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "gsi.h"
#define F(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  printf("gsi_query_opts %zu\n", sizeof(gsi_query_opts));
  printf("gsi_stats %zu\n", sizeof(gsi_stats));
  printf("gsi_graph_info %zu\n", sizeof(gsi_graph_info));
  printf("gsi_build_opts %zu\n", sizeof(gsi_build_opts));
  printf("gsi_buffer_desc %zu\n", sizeof(gsi_buffer_desc));
  F(gsi_query_opts, timeout_s) F(gsi_query_opts, stream) F(gsi_query_opts, n_roots)
  F(gsi_stats, count) F(gsi_stats, shard_row_end) F(gsi_stats, ms_kernel) F(gsi_stats, alg_bytes)
  F(gsi_stats, total_launches) F(gsi_graph_info, ms_build) F(gsi_graph_info, bytes_total)
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = subprocess.run([exe], capture_output=True, text=True).stdout
    return {l.split()[0]: int(l.split()[1]) for l in out.splitlines()}


def test_struct_layouts_match_header():
    c = _c_layout()
    assert c["gsi_query_opts"] == ctypes.sizeof(gsi.gsi_query_opts)
    assert c["gsi_stats"] == ctypes.sizeof(gsi.gsi_stats)
    assert c["gsi_graph_info"] == ctypes.sizeof(gsi.gsi_graph_info)
    assert c["gsi_build_opts"] == ctypes.sizeof(gsi.gsi_build_opts)
    assert c["gsi_buffer_desc"] == ctypes.sizeof(gsi.gsi_buffer_desc)
    for key, v in c.items():
        if "." in key:
            t, f = key.split(".")
            assert getattr(getattr(gsi, t), f).offset == v, key


@pytest.mark.skipif(gsi.gsi_device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_device_fails_loudly():
    g, q = W.fig1()
    with pytest.raises(gsi.GsiError) as e:
        gsi.build(g)
    assert e.value.status == "GSI_ERR_CUDA"
    assert "no CPU path" in str(e.value)


def test_query_signature_encoding_matches_oracle():
    for s in range(40):
        q = W.random_connected_query(s, 1 + s % 12, nlv=1 + s % 5, nle=1 + s % 7, extra=0.3)
        for distinct in (False, True):
            a = gsi.gsi_debug_query_signatures(q.vlabels, q.src, q.dst, q.elabels, distinct=distinct)
            b = oracle.query_signatures(q, distinct=distinct)
            assert np.array_equal(a, b), (s, distinct)


def test_invalid_arguments_are_errors():
    with pytest.raises(gsi.GsiError):
        gsi.gsi_debug_query_signatures(np.zeros(33), [], [], [])


def test_library_hashes_equal_known_answer_hashes():
    """The library's own hash code (host side of the __host__ __device__ functions its kernels
    call) against the oracle's general MurmurHash2 / MurmurHash64A, which are pinned to
    SMHasher's verification values in tests/test_oracle.py::test_murmur_known_answers.  A
    transcription slip shared by the device and the oracle specialisations would fail here."""
    rng = np.random.default_rng(12)
    for _ in range(300):
        x = int(rng.integers(0, 1 << 32))
        seed = int(rng.integers(0, 1 << 32))
        assert gsi.gsi_debug_hash(0, x, seed) == oracle.murmur2(x.to_bytes(4, "little"), seed)
        key = int(rng.integers(0, 1 << 62)) * 4 + int(rng.integers(0, 4))
        assert gsi.gsi_debug_hash(1, key, seed) == oracle.murmur64a(key.to_bytes(8, "little"), seed)
    # PCSR seeds are 0x9747B28C ^ label (reading A7)
    for l in range(5):
        assert gsi.gsi_debug_hash(0, 12345, 0x9747B28C ^ l) == oracle.murmur2((12345).to_bytes(4, "little"),
                                                                             0x9747B28C ^ l)

