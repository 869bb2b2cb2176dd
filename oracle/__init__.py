"""ORACLE TEST INFRASTRUCTURE (CPU checkers); see oracle/checkers.py."""
