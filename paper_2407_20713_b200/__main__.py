"""python -m paper_2407_20713_b200 {calibrate,eval,price,smile} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
