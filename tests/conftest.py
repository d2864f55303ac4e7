import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsrl.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    # Test-harness switch (the library itself reads no environment): a GPU test
    # re-run in a subprocess with SRL_TEST_TUNING="field=value,..." exercises an
    # opt-in kernel path through srl_set_tuning.
    spec = os.environ.get("SRL_TEST_TUNING")
    if spec:
        from paper_2603_23414_b200 import _lib
        _lib.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in spec.split(","))})
