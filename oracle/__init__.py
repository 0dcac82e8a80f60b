"""Parity oracle for the B200 decode path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

`attnkit_port` restates the reference's float64 decode path (attnkit/decode.py,
cache.py, latent.py, tpsim.py, zoo.py) in numpy. It is pinned to the reference by
golden vectors (`gen_golden.py` -> `tests/golden/`, checked in `tests/test_oracle.py`).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may
import this package, and only as the checker or the timed CPU baseline; the product
package `paper_2603_02188_b200` never imports it.

Parity status: PINNED -- the reference is pure Python and was imported in the dev
container to generate the golden vectors (`gen_golden.py`, committed).
"""
