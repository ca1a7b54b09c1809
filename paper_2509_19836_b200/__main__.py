"""``python -m paper_2509_19836_b200 {comm,balance,timeline}`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
