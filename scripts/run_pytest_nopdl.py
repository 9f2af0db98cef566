"""Run pytest with programmatic dependent launch disabled (diagnostics)."""
import sys

import pytest

sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), ".."))

from paper_2601_04707_b200._lib import lib

lib().mq_set_pdl(0)
sys.exit(pytest.main(sys.argv[1:]))
