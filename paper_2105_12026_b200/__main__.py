"""python -m paper_2105_12026_b200 summarize|surrogate ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
