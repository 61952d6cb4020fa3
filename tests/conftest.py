"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; the CPU suite runs with
-m "not gpu".  Golden fixtures were produced by running the reference
(tests/golden/make_golden.py); nothing here reads /root/reference."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def recombine_cases():
    return load_golden("recombine_cases.json")


@pytest.fixture(scope="session")
def factor_cases():
    return load_golden("factor_cases.json")


@pytest.fixture(scope="session")
def verify_cases():
    return load_golden("verify_cases.json")


@pytest.fixture(scope="session")
def big_inputs():
    return load_golden("big_inputs.json")


def rho_of(case):
    return [float.fromhex(h) for h in case["rho"]]


def poly_of(coeffs):
    from paper_2410_15880_b200 import IntPolynomial

    return IntPolynomial([int(c) for c in coeffs])
