import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# The loopback tests run up to 8 EP ranks x 2 micro-batches as threads of ONE
# process on ONE GPU, each on its own stream, with spin-waiting arrival
# kernels.  CUDA multiplexes streams onto CUDA_DEVICE_MAX_CONNECTIONS hardware
# queues (default 8): two ranks' streams sharing a queue would serialise a
# rank's signal behind another rank's wait.  One queue per stream (before the
# CUDA context exists).  One process per GPU -- the product setting -- uses
# two or three streams and is unaffected.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# ...and every kernel loaded when the context is created: with lazy loading
# (the CUDA 12 default) the first launch of a kernel waits for the kernels
# already running in the context, so one rank's first launch of, say, the
# arrival-signal kernel stalls behind another rank's spinning arrival wait
# until the wait times out (threads in one process only; separate processes
# have separate contexts).  The library refuses peer mode between ranks of one
# process under lazy loading (occ_comm_enable_peer).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
