"""Matrix Market texts shared by the golden generator (run against the
reference's io.load_matrix_market) and tests/test_mmio.py."""

GOOD = {
    "general_real": """%%MatrixMarket matrix coordinate real general
% a comment
%
4 5 7
1 1 1.5
2 3 -2.25e1
4 5 3.0
1 1 0.5
3 2 0

2 1 7
4 4 -1e-3
""",
    "integer_dups_cancel": """%%MatrixMarket matrix coordinate integer general
3 3 5
1 2 4
1 2 -4
2 2 9
3 1 -7
  3 3 1
""",
    "pattern_symmetric": """%%MatrixMarket matrix coordinate pattern symmetric
4 4 4
1 1
3 1
4 2
4 4
""",
    "real_symmetric": """%%MATRIXMARKET Matrix Coordinate Real Symmetric
3 3 4
1 1 2.0
2 1 -1.0
3 2 0.125
3 3 4.0
""",
    "empty": """%%MatrixMarket matrix coordinate real general
5 3 0
""",
}

BAD = {
    "bad_header": "%%MatrixMarket tensor coordinate real general\n1 1 0\n",
    "bad_field": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "bad_symmetry": "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    "array_layout": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "missing_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n3 three 1\n",
    "bad_entry": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 x 3.0\n",
    "missing_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 1.0\n",
    "too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 2.0\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 2.0\n",
}

# files that parse but whose canonical CSR holds a non-finite value: the
# reference's as_csr(coo, path) raises ValueError("<path> contains non-finite
# entries") (io.py:103, _validation.py:39-40)
NONFINITE = {
    "nonfinite_nan": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 nan\n",
    "nonfinite_inf": "%%MatrixMarket matrix coordinate real general\n2 3 2\n1 3 -inf\n2 2 2.0\n",
    "nonfinite_cancel": "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 inf\n1 2 -inf\n3 3 1.0\n",
}
