"""Generate the OSVD checkpoint fixtures (svd_layer.hpp:204-290) with the
UNMODIFIED reference (oracle/_ref): `make -C oracle && python tests/golden/make_osvd.py`.

  osvd_ref_6x4.bin   SvdParam::random(6, 4, 6, 4) (seed 3) + sigma ~ U(0.5, 2),
                     saved by save_svd_param_file: a reference-written file
  osvd_f32_5x7.bin   a parameter whose values are fp32-representable, saved by
                     the reference: the device round trip must reproduce it bit
                     for bit
Arrays of both are kept in osvd_golden.npz for the CPU-side checks.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402


def main():
    R = Ref()
    U, V, s, _, _ = R.gen_param(3, 6, 4, 6, 4, 1)
    R.svd_save(os.path.join(HERE, "osvd_ref_6x4.bin"), U, V, s, 6, 4)
    U2, V2, s2, _, _ = R.gen_param(4, 5, 7, 5, 3, 1)
    U2, V2, s2 = (a.astype(np.float32).astype(np.float64) for a in (U2, V2, s2))
    R.svd_save(os.path.join(HERE, "osvd_f32_5x7.bin"), U2, V2, s2, 5, 7)
    np.savez(os.path.join(HERE, "osvd_golden.npz"), ref_U=U, ref_V=V, ref_s=s, f32_U=U2, f32_V=V2, f32_s=s2)
    print("wrote osvd fixtures")


if __name__ == "__main__":
    main()
