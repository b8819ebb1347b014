"""Test-infrastructure oracle for the NSW ascent path (see nsw_oracle.py).

Never imported by the product package."""
