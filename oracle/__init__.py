"""Test infrastructure: CPU restatement (libhpo.so) and the reference compiled
from its own sources (oracle/_ref/). Never imported by the product path."""
