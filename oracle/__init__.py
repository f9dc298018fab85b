"""CPU oracle for arxiv 2005.13076's LeNet-style layer chain.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2005_13076_b200`` never imports it and
shares no code with it.
"""
