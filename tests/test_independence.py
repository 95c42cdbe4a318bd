"""CPU checks of the separation rules: the product package (paper_2406_14066_b200/) never imports,
links or executes oracle/ or the synthetic-input generator synth/, and the oracle never imports the
product.  The only module both sides use is synth/ (inputs), which holds none of the method's
arithmetic."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2406_14066_b200")
IMPORT = re.compile(r"^\s*(?:import|from)\s+(oracle|synth)\b", re.M)


def _sources(d, exts):
    for dp, _, fs in os.walk(d):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


def test_product_does_not_import_oracle_or_generator():
    bad = []
    for f in _sources(PKG, (".py",)):
        if IMPORT.search(open(f).read()):
            bad.append(os.path.relpath(f, ROOT))
    assert not bad, bad
    for f in _sources(os.path.join(PKG, "csrc"), (".cu", ".cuh", ".h")):
        assert not re.search(r'#include\s+"[^"]*oracle', open(f).read()), f


def test_oracle_does_not_import_product():
    for f in _sources(os.path.join(ROOT, "oracle"), (".py", ".c", ".h")):
        txt = open(f).read()
        assert not re.search(r"^\s*(?:import|from)\s+paper_2406_14066_b200\b", txt, re.M), f
        assert not re.search(r'#include\s+"[^"]*(tsv|csrc)', txt), f
        assert not re.search(r"^\s*(?:import|from)\s+synth\b", txt, re.M), f


def test_step_defaults_equal_generator_profiles():
    # the step's default latency profiles / seed are configuration duplicated on purpose (no import)
    import synth
    from paper_2406_14066_b200 import step
    assert step.DESK_TARGET == synth.SPEC_DESK_TARGET and step.DESK_DRAFT == synth.SPEC_DESK_DRAFT
    assert step.DEFAULT_SEED == synth.DEFAULT_SEED
