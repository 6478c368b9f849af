"""CPU-side checks of the C ABI: libchem.so loads (CUDA runtime present, no device needed) and
exports every symbol include/chem.h declares; the header and the binding agree; the product
package does not import the oracle.  No compute calls (there is no GPU here)."""
import ctypes
import pathlib
import re
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "chem.h").read_text()
    decl = re.findall(r"^\s*(?:int|void|size_t|const char\s*\*)\s+(chem_\w+)\s*\(", text, re.M)
    return sorted(set(decl))


def test_header_declarations_match_binding():
    from paper_2510_23993_b200 import binding
    assert sorted(binding.EXPORTED) == _declared()


def test_library_exports_every_symbol():
    from paper_2510_23993_b200 import binding, build
    build.build()
    lib = ctypes.CDLL(str(binding.LIB_PATH))
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(binding.LIB_PATH)], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_only():
    from paper_2510_23993_b200 import binding
    out = subprocess.run(["cuobjdump", "--list-elf", str(binding.LIB_PATH)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_default_opts_are_the_papers():
    from paper_2510_23993_b200 import binding
    o = binding.default_opts()
    # P:179 K_max = 5, P:181 N* (default < 0: one resident wave of the integration kernel)
    assert (o.kmax_bulk, o.n_active_star, o.kmax_sparse, o.T_min) == (5, -1, 100000, 500.0)
    assert (o.lockstep, o.kmax_first, o.compact_bulk, o.method) == (2, 1, 1, 0)
    # heavy-first schedule on cost hints: auto
    assert o.schedule_lpt == 2


def test_header_documents_the_defaults():
    """chem.h's comment of chem_default_opts states the values the library sets (VERDICT r01
    weak-6: it once said N* = 1e4 while the code set -1)."""
    import pathlib
    from paper_2510_23993_b200 import binding
    hdr = (pathlib.Path(__file__).resolve().parent.parent / "include" / "chem.h").read_text()
    doc = hdr[hdr.index("/* fills the defaults"):hdr.index("void chem_default_opts")]
    o = binding.default_opts()
    assert "n_active_star -1" in doc and o.n_active_star == -1
    assert "kmax_bulk 5" in doc and "kmax_sparse 1e5" in doc and "schedule_lpt 2" in doc
    assert "lockstep 2" in doc and "kmax_first 1" in doc and "T_min 500 K" in doc


def test_cell_status_rejects_unknown_workspace_without_gpu():
    """chem_cell_status on a workspace no call used is CHEM_EINVAL (checked before any device work)."""
    from paper_2510_23993_b200 import binding
    lib = binding.load_library()
    assert lib.chem_cell_status(None, None, 0, 0, 0, None, None, None) == -1


def test_opts_struct_matches_header():
    """The ctypes mirrors list the header's chem_opts / chem_stats fields in order (a missed field
    would shift every later one)."""
    import pathlib
    from paper_2510_23993_b200 import binding
    hdr = (pathlib.Path(__file__).resolve().parent.parent / "include" / "chem.h").read_text()
    for struct, cls in (("chem_opts", binding.ChemOpts), ("chem_stats", binding.ChemStats)):
        body = hdr[:hdr.index("} " + struct + ";")]
        body = body[body.rindex("typedef struct {"):]
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        names = re.findall(r"\b(\w+)(?:\[\d+\])?\s*[,;]", body)
        assert names == [n for n, _ in cls._fields_], (struct, names)


def test_init_rejects_unbalanced_mechanism_without_gpu():
    """chem_init validates before touching the device: an imbalanced row is CHEM_EMECH."""
    from paper_2510_23993_b200 import binding, mechanism
    lib = binding.load_library()
    mt = mechanism.load("toy_a_to_b")
    mt.nu_r[0, 1] = 2.0
    d, keep = binding.mech_desc(mt)
    h = ctypes.c_void_p()
    assert lib.chem_init(ctypes.byref(d), None, 0, ctypes.byref(h)) == -2


def test_init_unknown_structure_without_gpu():
    from paper_2510_23993_b200 import binding, mechanism
    lib = binding.load_library()
    mt = mechanism.load("toy_a_to_b")
    mt.reversible[0] = 1       # a reversible A<=>B with toy_a_to_b's numbers: valid, but the
    mt.A[0] = 7.0              # structure (reversible row) matches toy_a_eq_b -> accepted...
    d, keep = binding.mech_desc(mt)
    h = ctypes.c_void_p()
    rc = lib.chem_init(ctypes.byref(d), None, 0, ctypes.byref(h))
    assert rc in (0, -4)       # -4: structure matched but no CUDA device in this container
    mt.nu_f[0, 0] = 2.0        # 2A <=> 2B ... still balanced, no compiled structure
    mt.nu_r[0, 1] = 2.0
    d, keep = binding.mech_desc(mt)
    assert lib.chem_init(ctypes.byref(d), None, 0, ctypes.byref(h)) == -3


def test_product_does_not_import_oracle():
    code = ("import sys, paper_2510_23993_b200 as p; from paper_2510_23993_b200 import binding, mechanism, "
            "gen_structure, build; import paper_2510_23993_b200.api; "
            "assert not any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules), "
            "[m for m in sys.modules if 'oracle' in m]")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)


def test_no_oracle_reference_in_product_sources():
    for p in (ROOT / "paper_2510_23993_b200").rglob("*"):
        if p.suffix in (".py", ".cu", ".cuh", ".h"):
            txt = p.read_text()
            assert "import oracle" not in txt and "from oracle" not in txt, p
            assert "liboracle" not in txt, p
