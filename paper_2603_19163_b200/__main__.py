"""`python -m paper_2603_19163_b200 ...` (the reference's __main__.py:1-5)."""

import sys

from .cli import main

sys.exit(main())
