"""``python -m paper_2003_02547_b200`` -- the CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
