"""Seeded synthetic input generators (no method arithmetic). See synth.py."""
from . import synth  # noqa: F401
