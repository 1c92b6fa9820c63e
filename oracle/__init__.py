"""CPU oracle for the decode path -- TEST INFRASTRUCTURE ONLY.

Never imported by the product package; see ldpc_oracle.c for the parity pin.
"""
