"""python -m paper_2603_11868_b200 CASE [options] (see cli.py)"""
import sys

from .cli import main

sys.exit(main())
