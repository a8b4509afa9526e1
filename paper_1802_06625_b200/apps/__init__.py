"""Graph descriptions of the PRUNE applications the device executor runs."""
