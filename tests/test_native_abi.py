"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/mosaic_b200.h declares, and the ctypes table matches the header.
No kernel is launched (there is no GPU here)."""
import re
import subprocess

import pytest

from conftest import ROOT


def header_symbols():
    text = (ROOT / "include" / "mosaic_b200.h").read_text()
    return sorted(set(re.findall(r"MOSAIC_API\s+[\w\s\*]*?\b(mosaic_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for need in ("mosaic_mask_compact", "mosaic_gather_rows", "mosaic_lmhead_stats",
                 "mosaic_stats_merge", "mosaic_remask_commit", "mosaic_arena_reserve",
                 "mosaic_arena_commit", "mosaic_arena_release"):
        assert need in syms


def test_library_exports_every_header_symbol(native_lib):
    from paper_2601_06562_b200 import _native

    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (mosaic_\w+)", out))
    missing = set(header_symbols()) - exported
    assert not missing, missing
    assert set(_native.exported_symbols()) == set(header_symbols())


def test_library_loads_and_answers_host_queries(native_lib):
    from paper_2601_06562_b200 import _native, hotpath

    assert native_lib.mosaic_abi_version() == 100
    assert hotpath.mask_compact_scratch_bytes(1) == 4
    assert hotpath.mask_compact_scratch_bytes(4096 * 3 + 1) == 16
    assert hotpath.remask_scratch_bytes() >= 16 + 256 * 4
    del _native


def test_status_codes_map_to_reference_exceptions(native_lib):
    from paper_2601_06562_b200 import _native
    from paper_2601_06562_b200.errors import InputError

    # argument validation happens before any device work, so this runs on CPU
    with pytest.raises(InputError, match="multiple of 8"):
        _native.call("mosaic_gather_rows", None, 4, 3, 3, None, None, 0, 0, 0, None, None)
    with pytest.raises(InputError):
        _native.call("mosaic_stats_merge", None, None, None, 0, 1, None, 0, 1, None, None, None,
                     None, None, None, None)


def test_kernels_are_sm100a_tcgen05(native_lib):
    from paper_2601_06562_b200 import _native

    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True,
                          text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass, "LM head must issue tcgen05.mma"
    assert "UTMALDG" in sass, "operands must arrive through TMA"
    assert "LDTM" in sass, "epilogue must read TMEM with tcgen05.ld"
    elf = subprocess.run(["cuobjdump", "-lelf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in elf


def test_integration_stub_matches_the_abi():
    """The ctypes stub INTEGRATION.md tells a reference maintainer to add binds
    the same argument counts as this package's own binding (guards doc rot)."""
    import re

    from paper_2601_06562_b200 import _native

    text = (ROOT / "INTEGRATION.md").read_text()
    stub = text[text.index("for name, args in {"):text.index("}.items():")]
    entries = re.findall(r'"(mosaic_[a-z0-9_]+)":\s*\[(.*?)\],', stub, flags=re.S)
    assert len(entries) >= 6
    for name, args in entries:
        n_args = len([a for a in args.replace("\n", " ").split(",") if a.strip()])
        assert n_args == len(_native.SIGNATURES[name][1]), name
