import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# the engine's eigen-worker streams need more than CUDA's default 8 hardware queues (see
# paper_1612_07875_b200.recommended_env); set before any test initialises CUDA
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsdmd.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
