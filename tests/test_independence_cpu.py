"""Static checks of the separation the parity claims rest on:

- the product (`paper_2012_15198_b200/`, `include/`) never imports, includes or loads
  anything under `oracle/`, and the binding has no compute of its own (no numpy
  arithmetic on the hot path: it only marshals pointers);
- `oracle/` never imports the product or `synth/` (the shared input generators hold none
  of the method's arithmetic and are the only module both sides use);
- `synth/` imports neither side.
"""
import ast
import os
import re

from conftest import ROOT


def _py_imports(path):
    tree = ast.parse(open(path).read(), path)
    mods = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            mods.update(a.name.split(".")[0] for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.level == 0 and node.module:
            mods.add(node.module.split(".")[0])
    return mods


def _files(sub, exts):
    for dp, _, fns in os.walk(os.path.join(ROOT, sub)):
        for fn in fns:
            if fn.endswith(exts):
                yield os.path.join(dp, fn)


def test_product_never_touches_the_oracle():
    for f in _files("paper_2012_15198_b200", (".py",)):
        assert not (_py_imports(f) & {"oracle", "synth", "tests"}), f
        src = open(f).read()
        assert "oracle" not in re.sub(r'""".*?"""|#.*', "", src, flags=re.S), f
    for f in list(_files("paper_2012_15198_b200", (".cu", ".cuh", ".h", ".cpp"))) + list(_files("include", (".h",))):
        for inc in re.findall(r'#include\s*[<"]([^>"]+)[>"]', open(f).read()):
            assert "oracle" not in inc and "synth" not in inc, (f, inc)


def test_oracle_and_synth_never_touch_the_product():
    for f in _files("oracle", (".py",)):
        assert not (_py_imports(f) & {"paper_2012_15198_b200", "synth", "__graft_entry__", "torch"}), f
    for f in _files("synth", (".py",)):
        assert not (_py_imports(f) & {"paper_2012_15198_b200", "oracle", "__graft_entry__"}), f


def test_binding_only_marshals():
    src = open(os.path.join(ROOT, "paper_2012_15198_b200", "_lib.py")).read()
    code = re.sub(r'""".*?"""|#.*', "", src, flags=re.S)
    # no elementwise math on parameter data in Python: the only numpy use is host output arrays
    for forbidden in ("np.sqrt", "np.sum", ".sum(", "np.dot", " @ ", "torch.add", "torch.mul", ".mean("):
        assert forbidden not in code, forbidden
