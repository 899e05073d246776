"""ORACLE — test infrastructure only (see sdmd_oracle.py header).  Never imported by the
product package ``paper_1612_07875_b200``."""
from .sdmd_oracle import *  # noqa: F401,F403
from . import sdmd_oracle  # noqa: F401
