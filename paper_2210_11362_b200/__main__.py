"""`python -m paper_2210_11362_b200 ...` -- see cli.py."""

import sys

from .cli import main

sys.exit(main())
