"""Write the w10 empty-grating matrix as a column-major binary for tools/svd_probe."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "empty_w10.npz"))
A = z["A"]
with open(sys.argv[1], "wb") as fh:
    np.array(A.shape, dtype=np.int32).tofile(fh)
    np.asfortranarray(A).ravel(order="F").astype(np.complex128).tofile(fh)
