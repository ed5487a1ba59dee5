"""``python -m paper_2202_07258_b200 <gen|solve|bench|compare-t> ...`` (cli.py)."""

from .cli import main

main()
