"""Static check: no function in bench.py, __graft_entry__.py or the package
refers to a global name that is neither defined in its module, imported, nor
a builtin (a bench leg that only runs on the GPU box must not die of a
NameError there)."""

import builtins
import symtable
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
FILES = [ROOT / "bench.py", ROOT / "__graft_entry__.py",
         *sorted((ROOT / "paper_1901_10074_b200").glob("*.py")),
         *sorted((ROOT / "oracle").glob("*.py"))]


def _undefined(path):
    top = symtable.symtable(path.read_text(), str(path), "exec")
    module_names = {s.get_name() for s in top.get_symbols()
                    if s.is_assigned() or s.is_imported() or s.is_global() and s.is_assigned()}
    bad = []

    def walk(tab, chain):
        for sym in tab.get_symbols():
            name = sym.get_name()
            if sym.is_global() and not sym.is_assigned() and not sym.is_imported():
                if (name not in module_names and not hasattr(builtins, name)
                        and name not in ("__file__", "__name__", "__doc__")):
                    bad.append(f"{'.'.join(chain)}: {name}")
        for child in tab.get_children():
            walk(child, chain + [child.get_name()])

    walk(top, [path.name])
    return bad


@pytest.mark.parametrize("path", FILES, ids=lambda p: p.name)
def test_no_undefined_globals(path):
    assert _undefined(path) == []
