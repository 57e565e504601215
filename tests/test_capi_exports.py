"""CPU: the C-ABI library loads without a GPU, exports every symbol declared
in include/tierkv_b200.h, and the Python binding declares exactly those; the
product package never imports the oracle."""
import ctypes as ct
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tierkv_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tkv_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    names = declared_functions()
    for must in ["tkv_gather_layers", "tkv_scatter_layers", "tkv_hash_chains", "tkv_synth_pages",
                 "tkv_connector_get_num_new_matched_tokens", "tkv_connector_start_load_kv",
                 "tkv_connector_wait_load_kv", "tkv_connector_start_store_kv", "tkv_connector_wait_store_kv",
                 "tkv_connector_build_meta", "tkv_connector_update_state_after_alloc"]:
        assert must in names


def test_library_exports_every_declared_symbol(tkv):
    lib = ct.CDLL(tkv.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header(tkv):
    from paper_2510_09665_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == declared_functions()


def test_library_is_sm100a(tkv):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tkv.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_errc_names(tkv):
    lib = tkv.lib()
    assert lib.tkv_errc_name(0) == b"ok"
    assert lib.tkv_errc_name(2) == b"tier_full"
    assert lib.tkv_errc_name(16) == b"invalid_argument"


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2510_09665_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "tierkv_oracle" not in src and "libtierkv_ref" not in src, f
