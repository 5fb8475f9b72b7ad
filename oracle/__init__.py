"""CPU oracle for the quartic-K3 height path -- TEST INFRASTRUCTURE ONLY.

Loads oracle/_build/libqfs_oracle.so (plain C restatement of the reference
package, see qfs_oracle.c) through ctypes.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package;
the product package never does.
"""
from .oracle import *  # noqa: F401,F403
