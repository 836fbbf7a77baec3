"""`infersim` alias of the B200 package, so the reference's own tests
(/root/reference/pkg/tests, read-only) can run against it unchanged
(tests/test_reference_suite.py).  Test infrastructure only."""
from paper_2604_28175_b200 import *  # noqa: F401,F403
from paper_2604_28175_b200 import __version__  # noqa: F401
