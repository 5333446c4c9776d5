"""Test oracle (CPU). TEST INFRASTRUCTURE ONLY -- see oracle/oracle.py."""
