"""``python -m paper_2511_17361_b200 <command>``: the sqocc CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
