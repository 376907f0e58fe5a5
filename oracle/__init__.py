"""Test-infrastructure oracle (CPU restatement of the reference path).

Never imported by the product package; see cachetune_oracle.py header."""
