"""python -m paper_2605_11536_b200 <verb> ...: the tofr CLI on the B200 path (cli.py)."""
import sys

from .cli import main

sys.exit(main())
