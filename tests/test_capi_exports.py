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


def test_affine_form_host_rules():
    """tkv_affine_form (host only, no device work): consecutive chunks of one
    query have the form; a gap in the page columns, a second table, a short
    chunk before the last or uneven chunk spacing does not."""
    import ctypes as ct

    from paper_2510_09665_b200._lib import AffinePlanC, XferDescC, lib

    def descs(n=4, last=100, cs=1 << 20, fp_step=16, tables=None, short_at=None, bump_at=None):
        out = []
        for i in range(n):
            d = XferDescC(chunk=(1 << 30) + i * cs + (4096 if i == bump_at else 0), layer_stride=1 << 16, table_dev=(tables or [0x1000] * n)[i],
                          table_stride=512, first_page=3 + i * fp_step,
                          n_tokens=(last if i + 1 == n else (200 if i == short_at else 256)))
            out.append(d)
        return (XferDescC * n)(*out)

    def form(arr):
        p = AffinePlanC()
        rc = lib().tkv_affine_form(ct.cast(arr, ct.c_void_p), len(arr), 16, ct.byref(p))
        return rc, p
    rc, p = form(descs())
    assert rc == 0 and (p.n_desc, p.pages_per_desc, p.last_tokens, p.first_page) == (4, 16, 100, 3)
    assert p.chunk_stride == 1 << 20 and p.layer_stride == 1 << 16 and p.table_stride == 512
    rc, p = form(descs(n=1, last=256))
    assert rc == 0 and p.pages_per_desc == 16 and p.last_tokens == 256
    assert form(descs(fp_step=17))[0] != 0
    assert form(descs(tables=[0x1000, 0x1000, 0x2000, 0x1000]))[0] != 0
    assert form(descs(short_at=1))[0] != 0
    assert form(descs(last=0))[0] != 0
    assert form(descs(bump_at=2))[0] != 0
