"""CPU oracle package — test infrastructure only (checker + CPU baseline), never the product path."""
