"""``python -m paper_2604_04644_b200 bench ...`` (see cli.py)."""

import sys

from paper_2604_04644_b200.cli import main

sys.exit(main())
