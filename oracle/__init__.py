"""Parity oracle (TEST INFRASTRUCTURE): numpy restatement (veloreg_np) and the compiled
unmodified reference (ref -> oracle/_ref/libveloreg_ref.so).  Never imported by the product."""
