import sys

from paper_2601_13345_b200.cli import main

sys.exit(main())
