"""``python -m paper_1402_2020_b200 <subcommand>`` -- see cli.py."""
import sys

from .cli import main

sys.exit(main())
