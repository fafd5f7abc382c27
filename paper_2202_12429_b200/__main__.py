"""``python -m paper_2202_12429_b200 <subcommand>``: the embcache CLI over the B200 engine (cli.py)."""

import sys

from .cli import main

sys.exit(main())
