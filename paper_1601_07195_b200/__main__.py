"""``python -m paper_1601_07195_b200 <command>`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
