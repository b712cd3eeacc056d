"""python -m paper_2312_02376_b200 <solve|error-study|bench> ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
