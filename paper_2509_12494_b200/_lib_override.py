"""Experiment hook: tools/ scripts set PATH to an experiment build of the library before
importing paper_2509_12494_b200.ntt128.  None (the default) loads the in-tree product .so."""
PATH = None
