"""Stage the reference's own hot-path test files against this package (SURVEY
8(c) "Reusing the reference's tests against the build").

Run HERE (the container that has /root/reference): copies the reference
package and its tests into the git-ignored baseline/_ref/suite (gpurun ships
it to the GPU box) and writes a composite ``nenmf`` package whose hot-path
submodules (errors, matrix, nnls, compression, factorize, tracing) re-export
paper_1812_04315_b200, while the out-of-scope helpers the tests also import
(synthetic, CSV IO, host orthonormal_basis) come from the reference copy
``nenmf_ref``.  Then on the GPU box:

    bash baseline/_ref/suite/run.sh > gpurun_out/reference_suite.txt

Nothing of the reference is committed; the runner script and this stager are.
"""
import shutil
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg")
DST = REPO / "baseline" / "_ref" / "suite"
TESTS = ["test_nnls.py", "test_compression.py", "test_factorize.py", "test_matrix.py", "test_tracing.py",
         "test_synthetic.py", "test_cli.py", "test_acceptance.py"]
HOT = ["errors", "matrix", "nnls", "compression", "factorize", "tracing"]
# names a reference module exposes that live elsewhere in this package
EXTRA = {
    "matrix": "from nenmf_ref.matrix import QR_RANK_RTOL, orthonormal_basis, read_csv_matrix, write_csv_matrix\n"
              "from paper_1812_04315_b200.errors import RankDeficiencyError\n",
    "nnls": "from paper_1812_04315_b200.errors import NumericalFailureError\n"
            "from paper_1812_04315_b200.matrix import frobenius_norm, spectral_norm_sq\n",
    "compression": "from paper_1812_04315_b200.errors import NumericalCollapseError\n",
    "factorize": "from paper_1812_04315_b200.compression import compress_problem\n"
                 "from paper_1812_04315_b200.matrix import frobenius_norm\n"
                 "from paper_1812_04315_b200.nnls import solve_nnls\n",
    "tracing": "from pathlib import Path\nfrom paper_1812_04315_b200.matrix import frobenius_norm\n",
}


def main():
    if not REF.is_dir():
        sys.exit("no /root/reference here: stage in the build container")
    if DST.exists():
        shutil.rmtree(DST)
    (DST / "tests").mkdir(parents=True)
    shutil.copytree(REF / "src" / "nenmf", DST / "nenmf_ref", ignore=shutil.ignore_patterns("__pycache__"))
    for t in TESTS:
        shutil.copy(REF / "tests" / t, DST / "tests" / t)
    comp = DST / "nenmf"
    comp.mkdir()
    (comp / "__init__.py").write_text(
        "# composite: hot path from paper_1812_04315_b200, the rest from the reference copy;\n"
        "# the reference copy raises this package's exception classes\n"
        "import importlib\n"
        "import sys\n"
        "# the reference copy's hot-path submodules ARE this package's: its CLI and\n"
        "# generator then run on the GPU path (its host matrix helpers stay)\n"
        "for _m in ('errors', 'nnls', 'compression', 'factorize', 'tracing'):\n"
        "    sys.modules['nenmf_ref.' + _m] = importlib.import_module('paper_1812_04315_b200.' + _m)\n"
        "from paper_1812_04315_b200 import *  # noqa: F401,F403\n"
        "from nenmf_ref.matrix import orthonormal_basis, read_csv_matrix, write_csv_matrix  # noqa: F401\n"
        "from nenmf_ref.synthetic import ProblemInstance, generate_problem, load_instance, save_instance  # noqa\n")
    for m in HOT:
        (comp / f"{m}.py").write_text(f"from paper_1812_04315_b200.{m} import *  # noqa: F401,F403\n"
                                      + EXTRA.get(m, ""))
    (comp / "synthetic.py").write_text("from nenmf_ref.synthetic import *  # noqa: F401,F403\n"
                                       "from nenmf_ref.synthetic import generate_problem, load_instance, "
                                       "save_instance, ProblemInstance\n")
    (comp / "cli.py").write_text("from nenmf_ref.cli import *  # noqa: F401,F403\n"
                                 "from nenmf_ref.cli import derive_seed, main  # noqa: F401\n")
    (DST / "conftest.py").write_text(
        "# evidence that the suite ran through this package's CUDA library\n"
        "def pytest_sessionfinish(session, exitstatus):\n"
        "    from paper_1812_04315_b200 import _lib\n"
        "    lib = _lib.load_library()\n"
        "    print(f\"\\nlibnenmf_b200: {lib._name} kernel launches this session: {lib.nenmf_launch_count()}\")\n")
    (DST / "run.sh").write_text(
        "#!/bin/bash\n# the reference's hot-path tests against the composite package (GPU box)\n"
        "cd \"$(dirname \"$0\")\"\n"
        "PYTHONPATH=\"$PWD:$GRAFT_REPO_ROOT:${PYTHONPATH}\" python -m pytest tests -p no:cacheprovider "
        "-o addopts='' --rootdir=. \"$@\"\n")
    print("staged", DST)


if __name__ == "__main__":
    main()
