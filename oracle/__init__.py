"""Test-infrastructure oracle (reference CPU renderer wrapper)."""
