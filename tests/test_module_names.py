"""Every global name a package function refers to exists (a NameError on the
GPU-only paths would otherwise surface only on a B200 box)."""
import builtins
import importlib
import inspect
import types

import pytest

MODULES = ["paper_2410_15880_b200.verify", "paper_2410_15880_b200.recombine",
           "paper_2410_15880_b200.polynomial", "paper_2410_15880_b200.rootfinder",
           "paper_2410_15880_b200.parallel", "paper_2410_15880_b200.report",
           "paper_2410_15880_b200._lib"]


def _code_objects(code):
    yield code
    for c in code.co_consts:
        if isinstance(c, types.CodeType):
            yield from _code_objects(c)


@pytest.mark.parametrize("name", MODULES)
def test_functions_reference_defined_globals(name):
    mod = importlib.import_module(name)
    missing = []
    for fname, fn in vars(mod).items():
        if not inspect.isfunction(fn) or fn.__module__ != mod.__name__:
            continue
        for code in _code_objects(fn.__code__):
            # co_names holds globals, attributes and imports alike: check the
            # ones that are loaded as globals
            import dis

            for ins in dis.get_instructions(code):
                if ins.opname in ("LOAD_GLOBAL", "LOAD_NAME"):
                    g = ins.argval
                    if not hasattr(mod, g) and not hasattr(builtins, g):
                        missing.append((fname, g))
    assert not missing, missing
