"""``python -m paper_1408_5526_b200`` = the reference's ``python -m rqmcbench``."""
import sys

from .cli import main

sys.exit(main())
