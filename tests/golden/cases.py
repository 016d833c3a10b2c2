"""Engine parity case table shared by make_golden.py and the tests."""

ENGINE_CASES = [
    # (name, model, mode, codec, p, T, depth, warmup_epochs, lr, batch, decay_every)
    ("log_ds_none_p1", "log", "d_sync", 0, 1, 8, 2, 0, 0.2, 16, 0),
    ("log_ps_none_p1", "log", "pipe_sgd", 0, 1, 9, 2, 0, 0.15, 16, 0),
    ("log_ps_none_p1_k3", "log", "pipe_sgd", 0, 1, 9, 3, 0, 0.15, 16, 0),
    ("log_ds_t16_p2", "log", "d_sync", 1, 2, 7, 2, 0, 0.1, 16, 0),
    ("log_ps_q8_p4", "log", "pipe_sgd", 2, 4, 7, 2, 0, 0.1, 16, 0),
    ("mlp_ds_none_p4", "mlp", "d_sync", 0, 4, 6, 2, 0, 0.05, 25, 0),
    ("mlp_ps_none_p4", "mlp", "pipe_sgd", 0, 4, 6, 2, 0, 0.05, 25, 0),
    ("mlp_ps_t16_p2", "mlp", "pipe_sgd", 1, 2, 6, 2, 0, 0.05, 25, 3),
    ("mlp_ps_q8_p4", "mlp", "pipe_sgd", 2, 4, 6, 2, 0, 0.05, 25, 0),
    ("mlp_ds_q8_p2", "mlp", "d_sync", 2, 2, 6, 2, 0, 0.05, 25, 0),
    ("mlp_ps_t16_p4_warm", "mlp", "pipe_sgd", 1, 4, 12, 2, 1, 0.05, 32, 0),
    ("log_ps_q8_p1", "log", "pipe_sgd", 2, 1, 7, 2, 0, 0.1, 16, 0),
    ("log_pss_none_p1", "log", "ps_sync", 0, 1, 6, 2, 0, 0.2, 16, 0),
    ("mlp_pss_t16_p2", "mlp", "ps_sync", 1, 2, 6, 2, 0, 0.05, 25, 0),
    ("mlp_pss_q8_p4", "mlp", "ps_sync", 2, 4, 6, 2, 0, 0.05, 25, 3),
    ("log_pss_none_p4", "log", "ps_sync", 0, 4, 7, 2, 0, 0.1, 16, 0),
]
