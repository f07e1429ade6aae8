"""placeholder"""
LUFactors = factor_diagonal = factor_l_panel = factor_u_panel = factorize = residual = schur_update = solve = None
