"""Entry point: ``python -m paper_1112_5717_b200 <subcommand> ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
