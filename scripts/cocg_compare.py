import sys, numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
print("bitwise equal:", not bad, "differ:", bad)
for k in bad:
    print(k, np.linalg.norm(a[k] - b[k]) / np.linalg.norm(a[k]))
