"""TEST INFRASTRUCTURE ONLY: the CPU oracle package (parity checker and CPU baseline)."""
