import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# exactness claims of the oracle assume single-threaded BLAS
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")
# virtual ranks put several ranks' streams (5 each) in one CUDA context; with
# the default 8 hardware connections a stream-wait or spinning flag kernel of
# one rank can stall another rank's stream that shares its connection.  (Not
# for several processes sharing one GPU: tests/test_gpu_multiprocess.py and
# bench.py --share-gpu keep 8 — 32 per context stalled their handshake.)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run under gpurun)")
    config.addinivalue_line("markers", "slow: long CPU test")
