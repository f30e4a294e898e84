"""The C-ABI boundary: libsdp.so loads without a GPU, exports every function
include/sdp.h declares, and ctypes' struct layouts equal the C compiler's."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2507_09029_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sdp.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sdp_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    assert "sdp_owner_sync" in names and "sdp_build_masks" in names and len(names) >= 15


def test_library_exports_every_declared_symbol():
    lib = N.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers the whole header
    assert set(declared_functions()) == set(N.SIGNATURES)


def test_abi_version_and_error_string():
    lib = N.load()
    assert lib.sdp_abi_version() == N.ABI_VERSION
    assert isinstance(lib.sdp_last_error(), bytes)


def test_status_codes_map_to_reference_exceptions():
    from paper_2507_09029_b200 import errors as E
    lib = N.load()
    import ctypes as C
    # replication out of range is rejected before any device work
    words, nw = N.seed_words(1)
    rc = lib.sdp_assign_units(words, nw, None, 1, 1, 1, 4, 5, None, None, None)
    assert rc == 1
    with pytest.raises(E.ConfigError, match="replication"):
        N.check(rc)
    rc = lib.sdp_plan_tiles(None, 3, 10, 4096, None, None, None)
    with pytest.raises(E.ConfigError, match="mask_bytes"):
        N.check(rc)
    a = N.SyncArgs()
    a.dtype = 7
    with pytest.raises(E.ConfigError):
        N.check(lib.sdp_owner_sync(C.byref(a), None))
    with pytest.raises(E.UsageError):
        N.check(lib.sdp_ipc_close(C.c_void_p(1234)))


LAYOUT_C = r"""
#include <stdio.h>
#include <stddef.h>
#include "sdp.h"
#define F(S, f) printf(#S "." #f " %zu\n", offsetof(S, f));
int main(void) {
  printf("sdp_sync_args %zu\n", sizeof(sdp_sync_args));
  printf("sdp_tile_desc %zu\n", sizeof(sdp_tile_desc));
  printf("sdp_slice_desc %zu\n", sizeof(sdp_slice_desc));
  printf("sdp_param_desc %zu\n", sizeof(sdp_param_desc));
  printf("sdp_rule_desc %zu\n", sizeof(sdp_rule_desc));
  printf("sdp_group_desc %zu\n", sizeof(sdp_group_desc));
  F(sdp_sync_args, owner_mask) F(sdp_sync_args, replicas) F(sdp_sync_args, shadow_bf16)
  F(sdp_sync_args, lr) F(sdp_sync_args, status) F(sdp_sync_args, signal_pads)
  F(sdp_sync_args, epoch) F(sdp_sync_args, timeout_cycles) F(sdp_sync_args, epoch_counters)
  F(sdp_sync_args, slots) F(sdp_sync_args, slot_stride) F(sdp_sync_args, updates)
  F(sdp_sync_args, updates_per_cta) F(sdp_sync_args, states)
  printf("sdp_worker_state %zu\n", sizeof(sdp_worker_state));
  printf("sdp_update_desc %zu\n", sizeof(sdp_update_desc));
  F(sdp_slice_desc, rows) F(sdp_slice_desc, col_map) F(sdp_slice_desc, inner_shr)
  printf("sdp_slice_task %zu\n", sizeof(sdp_slice_task));
  printf("sdp_slice_segs %zu\n", sizeof(sdp_slice_segs));
  return 0;
}
"""


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(LAYOUT_C)
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True,
                                                              text=True, check=True).stdout.split("\n") if line)
    import ctypes as C
    assert int(out["sdp_sync_args"]) == C.sizeof(N.SyncArgs)
    assert int(out["sdp_tile_desc"]) == C.sizeof(N.TileDesc) == 16
    assert int(out["sdp_slice_desc"]) == C.sizeof(N.SliceDesc)
    assert int(out["sdp_param_desc"]) == C.sizeof(N.ParamDesc)
    assert int(out["sdp_rule_desc"]) == C.sizeof(N.RuleDesc)
    assert int(out["sdp_group_desc"]) == C.sizeof(N.GroupDesc)
    assert int(out["sdp_slice_task"]) == C.sizeof(N.SliceTask) == 32
    assert int(out["sdp_slice_segs"]) == C.sizeof(N.SliceSegs)
    assert int(out["sdp_worker_state"]) == C.sizeof(N.WorkerState) == 40
    assert int(out["sdp_update_desc"]) == C.sizeof(N.UpdateDesc) == 16
    from paper_2507_09029_b200.models import SLICE_DTYPE, TASK_DTYPE
    assert SLICE_DTYPE.itemsize == C.sizeof(N.SliceDesc) and TASK_DTYPE.itemsize == C.sizeof(N.SliceTask)
    for key, val in out.items():
        if "." in key:
            struct, field = key.split(".")
            cls = {"sdp_sync_args": N.SyncArgs, "sdp_slice_desc": N.SliceDesc}[struct]
            assert getattr(cls, field).offset == int(val), key
