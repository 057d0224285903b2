"""Argument lists of the CLI fixtures (shared by make_golden.py and tests/test_gpu_cli.py)."""

CLI_CASES = {
    "spatial": ["sphere-spatial", "--scheme", "LODIE1,AOSIE1", "--h", "0.5,0.25", "--T", "1.0"],
    "temporal": ["sphere-temporal", "--scheme", "LODIE2,MAOSIE", "--h", "0.25", "--dt",
                 "0.1,0.05,0.025", "--T", "0.5"],
    "stability": ["stability", "--scheme", "LODIE1,ExplicitEuler", "--h", "0.5", "--dt",
                  "0.01,0.1,1.0", "--T", "2.0"],
    "protein": ["protein", "--system", "SYS", "--h", "0.5", "--padding", "4", "--eps-m", "2",
                "--kappa-bar", "1.1283", "--variant", "Plain,RE,REplusV", "--dt", "0.5", "--T",
                "1.0", "--euler-dt", "0.002"],
    "vacuum": ["vacuum-check", "--system", "SYS", "--h", "0.5", "--padding", "4", "--eps-m",
               "2", "--dt", "0.5,0.25", "--T", "2.0"],
}
