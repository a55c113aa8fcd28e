import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def corpus():
    from tests.golden_corpus import load_corpus
    return load_corpus()


# LT_HANG_DUMP=1: SIGUSR1 dumps every thread's stack (diagnosing a process that
# does not exit, e.g. `timeout -s USR1 ... pytest`)
if os.environ.get("LT_HANG_DUMP"):
    import faulthandler
    import signal
    faulthandler.register(signal.SIGUSR1, all_threads=True, file=sys.__stderr__)
    # a C watchdog thread: dumps every Python thread and exits if the process is
    # still alive after LT_HANG_DUMP seconds (also during interpreter teardown)
    faulthandler.dump_traceback_later(float(os.environ["LT_HANG_DUMP"]), exit=True, file=sys.__stderr__)
