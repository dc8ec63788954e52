"""``python -m paper_1604_00617_b200 solve|verify|sweep|export ...`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
