"""The C-ABI library loads on a CPU-only host and exports every symbol
include/gravac_b200.h declares; struct layouts agree with the ctypes mirror."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2305_12201_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gravac_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"GVC_API\s+[\w\s\*]+?\b(gvc_\w+)\s*\(", src)))


def test_header_lists_match_binding():
    assert set(declared()) == set(_native.EXPORTS)


def test_library_exports_every_symbol():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2305_12201_b200 import build_ext
        build_ext.build()
    lib = _native.load()
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gvc_\w+)", out))
    assert set(declared()) <= exported
    assert lib.gvc_abi_version() == 2


def test_struct_layout_matches_c():
    # compile a tiny C probe against the header and compare sizeof/offsetof
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "gravac_b200.h"
int main(void){
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(gvc_select_result), offsetof(gvc_select_result, status),
         offsetof(gvc_select_result, kept_nonzero), sizeof(gvc_select_args),
         offsetof(gvc_select_args, dgc_sample_fraction), offsetof(gvc_select_args, force_exact));
  return 0;}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        vals = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    R, A = _native.SelectResult, _native.SelectArgs
    assert vals == [ctypes.sizeof(R), R.status.offset, R.kept_nonzero.offset, ctypes.sizeof(A),
                    A.dgc_sample_fraction.offset, A.force_exact.offset]


def test_argument_errors_without_gpu():
    lib = _native.load()
    args = _native.SelectArgs()
    args.kind = 7
    rc = lib.gvc_select(ctypes.byref(args), ctypes.c_void_p(16), 1 << 20, ctypes.c_void_p(16), None)
    assert rc == _native.GVC_ERR_ARG
    assert b"unknown compressor" in lib.gvc_last_error()
    args.kind = 0
    args.n = 0
    assert lib.gvc_select(ctypes.byref(args), ctypes.c_void_p(16), 1 << 20, ctypes.c_void_p(16), None) == \
        _native.GVC_ERR_ARG


def test_exchange_entry_points_validate_without_gpu():
    """The peer-exchange and DGC-sample entry points reject bad arguments
    before touching the device."""
    lib = _native.load()
    V = ctypes.c_void_p
    flags = (V * 9)(*([16] * 9))
    assert lib.gvc_peer_signal(flags, 9, 0, 1, None) == _native.GVC_ERR_ARG  # > GVC_MAX_PEERS ranks
    assert lib.gvc_peer_signal(flags, 2, 2, 1, None) == _native.GVC_ERR_ARG  # rank outside [0, nranks)
    assert lib.gvc_peer_signal(None, 2, 0, 1, None) == _native.GVC_ERR_ARG
    p2 = (V * 2)(16, 32)
    cnt = (ctypes.c_uint64 * 2)(4, 4)
    sg = _native.PeerStaging()
    sg.self_rank, sg.copy_blocks, sg.chunk_entries, sg.ready_dev = 0, 4, 1000, 16  # not a power of two
    for p in range(2):
        sg.src_idx_dev[p] = sg.src_vals_dev[p] = sg.src_bounds_dev[p] = 16
    assert lib.gvc_aggregate_peers_staged(p2, p2, p2, cnt, 2, 100, V(16), 1, ctypes.byref(sg), V(16), None) == \
        _native.GVC_ERR_ARG
    assert b"power of two" in lib.gvc_last_error()
    sg.chunk_entries, sg.self_rank = 1024, 5  # self outside the parts
    assert lib.gvc_aggregate_peers_staged(p2, p2, p2, cnt, 2, 100, V(16), 1, ctypes.byref(sg), V(16), None) == \
        _native.GVC_ERR_ARG
    assert lib.gvc_aggregate_peers(p2, p2, p2, cnt, 9, 100, V(16), 1, V(16), None) == _native.GVC_ERR_ARG
    assert lib.gvc_dgc_sample(100, 101, 0, 0, 0, V(16), None) == _native.GVC_ERR_ARG  # s > n
    assert lib.gvc_dgc_sample(100, 0, 0, 0, 0, V(16), None) == _native.GVC_ERR_ARG
    m = _native.EmitMirrors()
    m.count = 8  # more mirrors than peers
    assert lib.gvc_emit_mirrored(V(16), 1, 0, None, V(16), V(16), None, None, None, None, None, ctypes.byref(m),
                                 None) == _native.GVC_ERR_ARG


def test_exchange_struct_layouts_match_c():
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "gravac_b200.h"
int main(void){
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(gvc_emit_mirrors), offsetof(gvc_emit_mirrors, vals_dev),
         offsetof(gvc_emit_mirrors, bounds_dev), sizeof(gvc_peer_staging), offsetof(gvc_peer_staging, ready_dev),
         offsetof(gvc_peer_staging, src_vals_dev), offsetof(gvc_peer_staging, src_bounds_dev));
  return 0;}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(probe)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        vals = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    M, S = _native.EmitMirrors, _native.PeerStaging
    assert vals == [ctypes.sizeof(M), M.vals_dev.offset, M.bounds_dev.offset, ctypes.sizeof(S), S.ready_dev.offset,
                    S.src_vals_dev.offset, S.src_bounds_dev.offset]
