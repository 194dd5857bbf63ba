"""Build the oracle's native pieces (none yet beyond Python; placeholder
kept so __graft_entry__.build() has one entry point for checker code)."""


def build() -> None:
    return None
